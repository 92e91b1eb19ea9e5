# ncu --set full captures of the round-2 dominant kernels (one launch each)
set -x
O=gpurun_out/ncu
mkdir -p $O
DC="python bench.py --workload dcgan --B 32 --steps 1 --warmup 1 --no-graph --no-serial --no-cpu-baseline"
N="ncu --set full --clock-control none --import-source on --kernel-name-base demangled -c 1"
$N -k 'regex:k_gemm_tc<.bool.0, .bool.0, .int.256, .int.3, .bool.0, .bool.0, .int.0, .int.1>' -o $O/conv_fwd_s2 $DC > $O/a.log 2>&1
$N -k 'regex:k_gemm_tc<.bool.0, .bool.1, .int.64, .int.4, .bool.0, .bool.0, .int.0, .int.2>' -o $O/conv_dgrad_phase $DC > $O/b.log 2>&1
$N -k 'regex:k_gemm_tc<.bool.1, .bool.1, .int.128, .int.4, .bool.1, .bool.0, .int.0, .int.3>' -o $O/conv_wgrad $DC > $O/c.log 2>&1
$N -k 'regex:k_gemm_tf32x3<.bool.0, .bool.0, .int.128' -o $O/tf32_fwd python bench.py --dtype f32 --B 16 --steps 1 --warmup 1 --no-graph --no-serial --no-cpu-baseline > $O/d.log 2>&1
