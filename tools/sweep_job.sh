set -x
mkdir -p gpurun_out/sw
for w in pointnet_cls pointnet_seg dcgan; do
  timeout 900 python tools/sweep.py --workload $w --dtype bf16 --steps 5 --max-seconds 600 > gpurun_out/sw/sweep_${w}_bf16.jsonl 2> gpurun_out/sw/sweep_${w}_bf16.err
done
for w in pointnet_cls pointnet_seg dcgan; do
  timeout 900 python tools/sweep.py --workload $w --dtype f32 --steps 3 --Bs 1,2,4,8,16,32,64,128 --max-seconds 400 > gpurun_out/sw/sweep_${w}_f32.jsonl 2> gpurun_out/sw/sweep_${w}_f32.err
done
