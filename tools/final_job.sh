# Round-2 final measurement job (one gpurun call): the bench line of every
# workload, ncu launch lists with tensor-pipe activity and DRAM bytes, and
# ncu --set full captures of the dominant kernels.  Outputs: gpurun_out/final/.
set -x
O=gpurun_out/final
mkdir -p $O
python bench.py > $O/bench_cls_bf16.json 2> $O/bench_cls_bf16.err
python bench.py --workload pointnet_seg --no-serial --no-cpu-baseline > $O/bench_seg_bf16.json 2> $O/bench_seg_bf16.err
python bench.py --workload dcgan --no-serial --no-cpu-baseline > $O/bench_dcgan_bf16.json 2> $O/bench_dcgan_bf16.err
python bench.py --workload resnet18 --no-serial --no-cpu-baseline > $O/bench_resnet18_bf16.json 2> $O/bench_resnet18_bf16.err
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
DC="python bench.py --workload dcgan --B 32 --steps 1 --warmup 1 --no-graph --no-serial --no-cpu-baseline"
SG="python bench.py --workload pointnet_seg --B 32 --steps 1 --warmup 1 --no-graph --no-serial --no-cpu-baseline"
RS="python bench.py --workload resnet18 --B 64 --steps 1 --warmup 1 --no-graph --no-serial --no-cpu-baseline"
N="ncu --set full --clock-control none --import-source on --kernel-name-base demangled -c 1"
timeout 600 $N -k 'regex:k_gemm_tc<.bool.0, .bool.0, .int.32, .int.7, .bool.0, .bool.0, .int.0, .int.5' -o $O/conv_merged_phases $DC > $O/n1.log 2>&1
timeout 600 $N -k 'regex:k_gemm_tc<.bool.1, .bool.1, .int.256, .int.3, .bool.1, .bool.0, .int.0, .int.3' -o $O/conv_wgrad_256 $DC > $O/n2.log 2>&1
timeout 600 $N -k 'regex:k_bn_bwd_reduce_p' -o $O/bn_bwd_reduce_p $SG > $O/n3.log 2>&1
timeout 600 $N -k 'regex:k_bn_bwd_apply_p' -o $O/bn_bwd_apply_p $SG > $O/n4.log 2>&1
timeout 600 $N -k 'regex:k_gemm_tc<.bool.0, .bool.0, .int.64, .int.4, .bool.0, .bool.0, .int.0, .int.1, .bool.0' -o $O/resnet_conv_s1 $RS > $O/n5.log 2>&1
ls -la $O
