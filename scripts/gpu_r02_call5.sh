mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sharding.py tests/test_gpu_checked.py -q -m gpu > gpurun_out/c5_tests_a.log 2>&1; echo tests_a_rc=$?; tail -3 gpurun_out/c5_tests_a.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "variant or two_kernel or cached or lean" > gpurun_out/c5_tests_b.log 2>&1; echo tests_b_rc=$?; tail -3 gpurun_out/c5_tests_b.log
AB_REPS=3 timeout 600 python scripts/ab_options.py C4:c64 -- tile_schedule=2 variant=1 variant=3 > gpurun_out/ab_c5.jsonl 2>&1; cat gpurun_out/ab_c5.jsonl
PROXY_STEPS=20 timeout 900 python scripts/loopback_proxy.py > gpurun_out/loopback_proxy_fused.jsonl 2>&1; cat gpurun_out/loopback_proxy_fused.jsonl
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log
