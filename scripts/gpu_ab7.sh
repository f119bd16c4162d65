timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharding.py -q -m gpu -x --timeout 200 2>&1 | tail -2
for rep in 1 2 3; do
  timeout 120 python scripts/sweep_cfg.py C4 c64 20 2>&1 | tail -1 | sed "s/^/rev /"
  NLSE_NO_REV=1 timeout 120 python scripts/sweep_cfg.py C4 c64 20 2>&1 | tail -1 | sed "s/^/norev /"
  timeout 120 python scripts/sweep_cfg.py C5W c128 20 2>&1 | tail -1 | sed "s/^/rev5 /"
  NLSE_NO_REV=1 timeout 120 python scripts/sweep_cfg.py C5W c128 20 2>&1 | tail -1 | sed "s/^/norev5 /"
  timeout 120 python scripts/sweep_cfg.py C3 c128 20 2>&1 | tail -1 | sed "s/^/rev3 /"
  NLSE_NO_REV=1 timeout 120 python scripts/sweep_cfg.py C3 c128 20 2>&1 | tail -1 | sed "s/^/norev3 /"
done
