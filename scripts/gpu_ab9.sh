timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharding.py tests/test_gpu_schemes.py -q -m gpu -x --timeout 200 2>&1 | tail -1
for rep in 1 2; do
  timeout 120 python scripts/sweep_cfg.py C4 c64 20 2>&1 | tail -1 | sed "s/^/C4 /"
  timeout 120 python scripts/sweep_cfg.py C5W c128 20 2>&1 | tail -1 | sed "s/^/C5Wd /"
  timeout 120 python scripts/sweep_cfg.py C5W c64 20 2>&1 | tail -1 | sed "s/^/C5Wf /"
  timeout 120 python scripts/sweep_cfg.py C3 c128 20 2>&1 | tail -1 | sed "s/^/C3 /"
done
