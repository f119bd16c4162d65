timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharding.py -q -m gpu --timeout 120 -x > gpurun_out/gpu_all.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/gpu_all.log
for rep in 1 2; do echo "$(timeout 300 python scripts/sweep.py 2>&1 | tail -1)"; done
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_q.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu_rc=$?
