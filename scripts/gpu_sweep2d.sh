# 2D preset sweep: C3 8192^2 in c128 and c64 with each build/lib_p*.so
for rep in 1 2; do
for p in ${PRESETS:-0 1 2 3}; do
  for dt in c128 c64; do
    NLSE_LIB=build/lib_p$p.so timeout 120 python scripts/sweep_cfg.py C3 $dt 20 2>&1 | tail -1
  done
done
done
