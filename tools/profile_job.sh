# Round-2 measurement job (one gpurun call): bench lines of every workload at
# its sweep peak, launch lists with tensor-pipe activity, ncu --set full
# captures of the dominant kernels.  Outputs under gpurun_out/prof/.
set -x
O=gpurun_out/prof
mkdir -p $O
python bench.py > $O/bench_cls_bf16.json 2> $O/bench_cls_bf16.err
python bench.py --workload pointnet_seg --no-serial --no-cpu-baseline > $O/bench_seg_bf16.json 2> $O/bench_seg_bf16.err
python bench.py --workload dcgan --no-serial --no-cpu-baseline > $O/bench_dcgan_bf16.json 2> $O/bench_dcgan_bf16.err
python bench.py --dtype f32 --steps 3 --no-serial --no-cpu-baseline > $O/bench_cls_f32.json 2> $O/bench_cls_f32.err
python bench.py --workload dcgan --dtype f32 --steps 3 --no-serial --no-cpu-baseline > $O/bench_dcgan_f32.json 2> $O/bench_dcgan_f32.err
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum
for w in pointnet_cls pointnet_seg dcgan; do
  B=64; [ $w = dcgan ] && B=32
  ncu --metrics $M --clock-control none --csv --log-file $O/launches_${w}_b${B}.csv \
      python bench.py --workload $w --B $B --steps 1 --warmup 1 --no-graph --no-serial --no-cpu-baseline > $O/ncu_${w}.log 2>&1
done
