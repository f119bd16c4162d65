# A/B: default build vs build/lib_old.so on the 3D configs
for rep in 1 2; do
for cfg in "C4 c64" "C5W c128"; do
  timeout 120 python scripts/sweep_cfg.py $cfg 20 2>&1 | tail -1
  NLSE_LIB=build/lib_old.so timeout 120 python scripts/sweep_cfg.py $cfg 20 2>&1 | tail -1
done
done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x --timeout 120 -k "3-" 2>&1 | tail -2
