for lib in ${LIBS}; do
  NLSE_VARIANT=4 NLSE_LIB=$lib timeout 120 python scripts/sweep_cfg.py C4 c64 10 2>&1 | tail -1
done
