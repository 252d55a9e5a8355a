for v in variants/w_c32u4.so variants/w_c32u8.so variants/w_c64u4.so variants/w_c64u8.so variants/w_c16u16.so variants/w_c32u4.so; do
  echo "== $v"; UCP_B200_LIB=$v python tools/profile_step.py --log2d 18 --phases exh0,local0 --steps 3 --warmup 1 2>&1 | tail -3
done > gpurun_out/walk_variants2.log 2>&1
cat gpurun_out/walk_variants2.log
