# round 2: full GPU suite with the parity log, then the bench (run under gpurun)
mkdir -p gpurun_out
nproc; free -g | head -2; nvidia-smi --query-gpu=name,memory.total,clocks.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
tail -2 gpurun_out/smoke.log
rm -f gpurun_out/parity_r02.jsonl
PARITY_LOG=$PWD/gpurun_out/parity_r02.jsonl timeout 1700 python -m pytest tests -q -m gpu --durations=40 > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$?
tail -60 gpurun_out/gpu_tests.log
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo bench_rc=$?
tail -1 gpurun_out/bench.log
