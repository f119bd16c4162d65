timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_schemes.py tests/test_gpu_sharding.py -q -m gpu -x -k "variant or two_kernel or fused_and_two or switch or loopback_bitwise" > gpurun_out/c17_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/c17_tests.log
AB_REPS=3 timeout 900 python scripts/ab_options.py C4:c64 C3:c128 -- variant=1 variant=3 > gpurun_out/ab_c17.jsonl 2>&1; cut -c1-125 gpurun_out/ab_c17.jsonl
timeout 900 ncu --set full --clock-control none -k regex:two_ --launch-count 2 -o gpurun_out/two_kernel2 -f python scripts/one_step.py C4 c64 1 variant=1 > /dev/null 2>&1; echo ncu=$?
python scripts/ncu_summary.py gpurun_out/two_kernel2.ncu-rep | grep -v "^   [a-z]*__[a-z_]*\.sum  *[0-9]" | head -30
