mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharding.py -q -m gpu -x -k "not C5S and not C5W and not fig" > gpurun_out/c3_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/c3_tests.log
timeout 300 python scripts/call_overhead.py > gpurun_out/call_overhead.jsonl 2>&1; cat gpurun_out/call_overhead.jsonl
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo bench_rc=$?; tail -1 gpurun_out/bench.log
timeout 300 python bench.py --steps 20 --warmup 5 --workload C5W --no-cpu-baseline > gpurun_out/bench_c5w.log 2>&1; tail -1 gpurun_out/bench_c5w.log
