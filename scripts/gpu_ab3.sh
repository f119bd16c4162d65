timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharding.py tests/test_gpu_schemes.py -q -m gpu -x --timeout 200 2>&1 | tail -3
for rep in 1 2; do
for cfg in "C4 c64" "C3 c128" "C5W c128"; do
  timeout 120 python scripts/sweep_cfg.py $cfg 20 2>&1 | tail -1
  NLSE_LIB=build/lib_old.so timeout 120 python scripts/sweep_cfg.py $cfg 20 2>&1 | tail -1
done
done
