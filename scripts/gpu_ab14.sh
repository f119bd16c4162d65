for rep in 1 2 3; do
for lib in build/lib_a00.so build/lib_a10.so build/lib_a01.so paper_1109_1027_b200/libnlse2shoc.so; do
  NLSE_LIB=$lib timeout 120 python scripts/sweep_cfg.py C4 c64 20 2>&1 | tail -1
  NLSE_LIB=$lib timeout 120 python scripts/sweep_cfg.py C5W c128 20 2>&1 | tail -1
done
done
