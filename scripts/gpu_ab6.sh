for rep in 1 2 3; do
for pp in 256 128 64 0; do
  NLSE_TMA_PROMO_P=$pp timeout 120 python scripts/sweep_cfg.py C4 c64 20 2>&1 | tail -1 | sed "s/^/C4_pp=$pp /"
done
for pr in 0 64; do
  NLSE_TMA_PROMO=$pr timeout 120 python scripts/sweep_cfg.py C5W c128 20 2>&1 | tail -1 | sed "s/^/C5Wd_pr=$pr /"
  NLSE_TMA_PROMO=$pr timeout 120 python scripts/sweep_cfg.py C3 c128 20 2>&1 | tail -1 | sed "s/^/C3_pr=$pr /"
done
done
