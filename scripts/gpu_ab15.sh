for rep in 1 2; do
for lib in paper_1109_1027_b200/libnlse2shoc.so build/lib_p3.so build/lib_p6.so build/lib_p0.so; do
  NLSE_LIB=$lib timeout 120 python scripts/sweep_cfg.py C3 c128 20 2>&1 | tail -1
  NLSE_LIB=$lib timeout 120 python scripts/sweep_cfg.py C3 c64 20 2>&1 | tail -1
done
done
