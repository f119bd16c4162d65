for rep in 1 2 3; do
for lib in build/lib_r0.so build/lib_r4.so build/lib_r5.so build/lib_r6.so; do
  NLSE_LIB=$lib timeout 120 python scripts/sweep_cfg.py C4 c64 20 2>&1 | tail -1
done
done
