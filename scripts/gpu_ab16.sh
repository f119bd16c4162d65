for rep in 1 2 3; do
for lib in paper_1109_1027_b200/libnlse2shoc.so build/lib_d32.so build/lib_d40.so build/lib_d36.so build/lib_d32n16.so; do
  NLSE_LIB=$lib timeout 120 python scripts/sweep_cfg.py C5W c128 20 2>&1 | tail -1
done
done
