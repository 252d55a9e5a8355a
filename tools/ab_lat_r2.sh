for v in default variants/lat6.so variants/lat4.so variants/lat2.so; do
  if [ $v = default ]; then L=""; else L="UCP_B200_LIB=$v"; fi
  echo "== $v"
  env $L python tools/shard_projection.py --ns 1 8 2>&1 | python -c "import json,sys; [print(json.dumps({k: d[k] for k in ('n_gpus','projected_step_ms','efficiency_vs_1','phase_ms_max_over_ranks','imbalance_max_over_mean')})) for d in map(json.loads, sys.stdin)]"
  env $L python tools/c1_latency.py --n 5 --modes fresh 2>&1 | cut -c1-120
  env $L python tools/converge.py --d 14000 2>&1 | tail -1 | cut -c1-100
done > gpurun_out/lat_variants.log 2>&1
cat gpurun_out/lat_variants.log
