for rep in 1 2; do
for lib in ${LIBS}; do
  NLSE_LIB=$lib timeout 120 python scripts/sweep_cfg.py C4 c64 20 2>&1 | tail -1
done
done
