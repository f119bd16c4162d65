for rep in 1 2; do
for lib in paper_1109_1027_b200/libnlse2shoc.so build/lib_f24.so build/lib_f24r4.so build/lib_f32r2.so; do
  NLSE_LIB=$lib timeout 120 python scripts/sweep_cfg.py C4 c64 20 2>&1 | tail -1
done
done
