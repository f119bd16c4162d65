# quick iteration: parity tests, then bench, then a launch-list ncu pass
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 120 -x > gpurun_out/gpu_all.log 2>&1; echo tests_rc=$?; tail -4 gpurun_out/gpu_all.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
if [ "$NCU" = "1" ]; then
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu1.log 2>&1; echo ncu1_rc=$?
fi
if [ "$NCUFULL" = "1" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stage_stream -s 12 -c 4 -o gpurun_out/prof_c4 -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu2.log 2>&1; echo ncu2_rc=$?
fi
