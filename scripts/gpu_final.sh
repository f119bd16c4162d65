# Round measurement: smoke, GPU suite (slow tests on), bench (both arms), launch list, one
# --set full capture of the C4 stage kernels, perf table.  Outputs under gpurun_out/.
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
NLSE_SLOW=1 timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_all.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/gpu_all.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
timeout 600 python bench.py --impl reference > gpurun_out/bench_reference.json 2> gpurun_out/bench_ref.err; echo ref_rc=$?
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu1_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stage_stream -s 12 -c 4 -o gpurun_out/prof_c4 -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu2.log 2>&1; echo ncu2_rc=$?
timeout 900 python scripts/perf_table.py > gpurun_out/perf_table.jsonl 2>&1; echo perf_rc=$?
