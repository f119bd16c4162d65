# HEAD verification on a B200 (under gpurun); outputs in gpurun_out/
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/s3_gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3_smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/s3_smoke.log
rm -f gpurun_out/s3_parity.jsonl
PARITY_LOG=$PWD/gpurun_out/s3_parity.jsonl timeout 1500 python -m pytest tests -q -m gpu --durations=12 > gpurun_out/s3_tests.log 2>&1; echo tests_rc=$?; tail -22 gpurun_out/s3_tests.log
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/s3_bench.json 2> gpurun_out/s3_bench.err; echo bench_rc=$?; cat gpurun_out/s3_bench.json | cut -c1-600
timeout 300 python bench.py --steps 20 --warmup 5 --workload C5W --no-cpu-baseline > gpurun_out/s3_bench_c5w.json 2>&1; tail -1 gpurun_out/s3_bench_c5w.json | cut -c1-300
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file gpurun_out/s3_launches_C4.csv python scripts/one_step.py C4 c64 2 > /dev/null 2>&1; echo ncu_rc=$?
python scripts/launches.py gpurun_out/s3_launches_C4.csv 452984832 | tee gpurun_out/s3_launches_C4_summary.txt
