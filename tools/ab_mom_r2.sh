for v in ${VARIANTS:-default variants/m_u8b4.so variants/m_u4b8.so variants/m_u2b8.so variants/m_u8b3.so default}; do
  if [ $v = default ]; then L=""; else L="UCP_B200_LIB=$v"; fi
  echo "== $v"; env $L python tools/profile_step.py --log2d 18 --phases local1 --steps 3 --warmup 1 2>&1 | tail -3
done > gpurun_out/${OUT:-mom_variants}.log 2>&1
cat gpurun_out/${OUT:-mom_variants}.log
