for v in default variants/fq4p6.so variants/fq8p6.so variants/fq4p8.so variants/fq8p14.so default; do
  if [ $v = default ]; then L=""; else L="UCP_B200_LIB=$v"; fi
  echo "== $v"
  env $L python tools/c1_latency.py --n 7 --modes fresh 2>&1 | cut -c1-110
  env $L python tools/moments_sweep.py 2000 6000 8192 2>&1 | tail -3 | tr '\n' ' '; echo
done > gpurun_out/fused_variants.log 2>&1
cat gpurun_out/fused_variants.log
