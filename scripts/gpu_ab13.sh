for rep in 1 2 3; do
for lib in paper_1109_1027_b200/libnlse2shoc.so build/lib_l2.so build/lib_l1.so build/lib_l8.so; do
  NLSE_LIB=$lib timeout 120 python scripts/sweep_cfg.py C2 c128 50 2>&1 | tail -1
  NLSE_LIB=$lib timeout 120 python scripts/sweep_cfg.py C2 c64 50 2>&1 | tail -1
done
done
