for v in default variants/q64b4.so variants/q64b3.so variants/q32b8.so; do
  if [ $v = default ]; then L=""; else L="UCP_B200_LIB=$v"; fi
  echo "== $v"
  env $L python tools/shard_projection.py --ns 1 8 2>&1 | python -c "import json,sys; [print(d['n_gpus'], round(d['projected_step_ms'],1), round(d['efficiency_vs_1'],4), d['phase_ms_max_over_ranks']['local1'], [r[1] for r in d['rank_phase_ms']]) for d in map(json.loads, sys.stdin)]"
  env $L python tools/profile_step.py --log2d 18 --phases local1 --steps 2 --warmup 1 | tail -1
done > gpurun_out/momqt_variants.log 2>&1
cat gpurun_out/momqt_variants.log
