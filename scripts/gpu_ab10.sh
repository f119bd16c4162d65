timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 100 -k "1- or msd or C2" 2>&1 | tail -1
for rep in 1 2 3; do
for dt in c128 c64; do
  timeout 120 python scripts/sweep_cfg.py C2 $dt 50 2>&1 | tail -1 | sed "s/^/rev_$dt /"
  NLSE_NO_REV=1 timeout 120 python scripts/sweep_cfg.py C2 $dt 50 2>&1 | tail -1 | sed "s/^/norev_$dt /"
done
done
