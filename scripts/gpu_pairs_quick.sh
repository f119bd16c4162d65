timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 60 -k "rk4_parity_10_steps and -4]" 2>&1 | tail -2
for cfg in "C4 c64" "C3 c128" "C5W c128"; do
  for v in ${VARIANTS:-0 4}; do NLSE_VARIANT=$v timeout 120 python scripts/sweep_cfg.py $cfg 20 2>&1 | tail -1; done
done
