# stage-pair (variant 4) vs per-stage (variant 0) timing on the BASELINE grids
for rep in 1 2; do
for cfg in "C4 c64" "C3 c128" "C3 c64" "C5W c64" "C5W c128"; do
  for v in 0 4; do NLSE_VARIANT=$v timeout 120 python scripts/sweep_cfg.py $cfg 20 2>&1 | tail -1; done
done
done
