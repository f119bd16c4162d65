timeout 900 python -m pytest tests -q -m gpu -x -k "not C5S and not C5W and not C2_full and not C3_full and not fig" > gpurun_out/c9_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/c9_tests.log
timeout 300 python scripts/one_step.py C4 c64 1 variant=1 > /dev/null 2>&1; echo plain=$?
timeout 900 ncu --set full --clock-control none -k regex:two_ --launch-count 4 -o gpurun_out/two_kernel -f python scripts/one_step.py C4 c64 1 variant=1 > gpurun_out/ncu_two.log 2>&1; echo ncu_two=$?
python scripts/ncu_summary.py gpurun_out/two_kernel.ncu-rep
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log
