# Round-2 final measurement job (one gpurun call): the bench line of every
# workload (twice for the headline workloads: box-to-box spread), the
# reference arm, ncu launch lists with tensor-pipe activity and DRAM bytes.
# Outputs: gpurun_out/final7/.
set -x
O=gpurun_out/final7
mkdir -p $O
python bench.py > $O/bench_cls_bf16.json 2> $O/bench_cls_bf16.err
python bench.py --no-serial --no-cpu-baseline > $O/bench_cls_bf16_b.json 2> $O/bench_cls_bf16_b.err
for w in pointnet_seg dcgan resnet18; do
  python bench.py --workload $w --no-serial --no-cpu-baseline > $O/bench_${w}_bf16.json 2> $O/bench_${w}_bf16.err
  python bench.py --workload $w --no-serial --no-cpu-baseline > $O/bench_${w}_bf16_b.json 2> $O/bench_${w}_bf16_b.err
done
python bench.py --dtype f32 --steps 3 --no-serial --no-cpu-baseline > $O/bench_cls_f32.json 2> $O/bench_cls_f32.err
python bench.py --workload dcgan --dtype f32 --steps 3 --no-serial --no-cpu-baseline > $O/bench_dcgan_f32.json 2> $O/bench_dcgan_f32.err
python bench.py --workload resnet18 --dtype f32 --steps 3 --no-serial --no-cpu-baseline > $O/bench_resnet18_f32.json 2> $O/bench_resnet18_f32.err
python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum
for w in pointnet_cls pointnet_seg dcgan resnet18; do
  B=64; [ $w = dcgan ] && B=32
  timeout 900 ncu --metrics $M --clock-control none --csv --log-file $O/launches_${w}_b${B}.csv \
      python bench.py --workload $w --B $B --steps 1 --warmup 1 --no-graph --no-serial --no-cpu-baseline > $O/ncu_${w}.log 2>&1
done
ls -la $O
