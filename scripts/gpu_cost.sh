# new-option test, live kernel timeline, and the measured counterpart of the paper's Tables 3-5
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "check_every or caller_owned or padded_layout or carried_sum" > gpurun_out/opt_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/opt_tests.log
for a in "C4 c64 20" "C4 c64 100" "C4 c64 20 cuda_graph=0" "C5W c128 20"; do timeout 300 python scripts/timeline.py $a >> gpurun_out/timeline.jsonl 2>> gpurun_out/timeline.err; done; cut -c1-900 gpurun_out/timeline.jsonl
timeout 1200 python scripts/cost_tables.py --steps 10 > gpurun_out/cost_time_v2.jsonl 2> gpurun_out/cost_time_v2.err; echo cost_time_rc=$?
timeout 1800 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/cost_launches_v2.csv python scripts/cost_tables.py --ncu > gpurun_out/cost_ncu_run_v2.log 2>&1; echo cost_ncu_rc=$?
grep "^ORDER " gpurun_out/cost_ncu_run_v2.log | sed 's/^ORDER //' > gpurun_out/cost_order_v2.json
python scripts/cost_tables.py --parse gpurun_out/cost_launches_v2.csv gpurun_out/cost_order_v2.json > gpurun_out/cost_ncu_v2.jsonl
python scripts/cost_tables.py --report gpurun_out/cost_time_v2.jsonl gpurun_out/cost_ncu_v2.jsonl MEASURED_PEAKS.json | tee gpurun_out/cost_tables_v2.md | head -24
gzip -f gpurun_out/cost_launches_v2.csv
