timeout 900 python -m pytest tests -q -m gpu --timeout 300 -k "3-" 2>&1 | tail -1
for rep in 1 2; do
for lib in paper_1109_1027_b200/libnlse2shoc.so build/lib_f32.so; do
  NLSE_LIB=$lib timeout 120 python scripts/sweep_cfg.py C4 c64 20 2>&1 | tail -1
done
done
