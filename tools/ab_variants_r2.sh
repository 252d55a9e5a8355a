set -x
for v in default variants/w_u4.so variants/w_u1.so variants/w_c32.so variants/w_c32u4.so variants/w_mb10.so variants/w_mb14.so default; do
  if [ $v = default ]; then L=""; else L="UCP_B200_LIB=$v"; fi
  echo "== $v"; env $L python tools/profile_step.py --log2d 18 --phases exh0,local0 --steps 3 --warmup 1 2>&1 | tail -3
done > gpurun_out/walk_variants.log 2>&1
for v in default variants/unifold.so default; do
  if [ $v = default ]; then L=""; else L="UCP_B200_LIB=$v"; fi
  echo "== $v"; env $L python tools/bench_config5.py --cpu-rounds 0 --cases zd_2000,zd_16384,inv3_601,inv8_601,inv3_4096 2>&1 | tail -5
done > gpurun_out/c5_variants.log 2>&1
python -m pytest tests/test_gpu_config5.py tests/test_gpu_kernels_module.py tests/test_gpu_stress.py -x -q > gpurun_out/c5_tests.log 2>&1; echo rc=$? >> gpurun_out/c5_tests.log
tail -3 gpurun_out/c5_tests.log
