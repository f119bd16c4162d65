mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x --durations=15 > gpurun_out/c11_tests.log 2>&1; echo tests_rc=$?; tail -20 gpurun_out/c11_tests.log
timeout 900 python scripts/cost_tables.py > gpurun_out/cost_time.jsonl 2> gpurun_out/cost_time.err; echo cost_rc=$?
timeout 900 python scripts/cost_tables.py --ncu > gpurun_out/cost_order.txt 2>&1; echo plain_rc=$?
grep '^ORDER ' gpurun_out/cost_order.txt | sed 's/^ORDER //' > gpurun_out/cost_order.json
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/cost_launches.csv python scripts/cost_tables.py --ncu > /dev/null 2>&1; echo ncu_rc=$?
python scripts/cost_tables.py --parse gpurun_out/cost_launches.csv gpurun_out/cost_order.json > gpurun_out/cost_ncu.jsonl; echo parse_rc=$?
python scripts/cost_tables.py --report gpurun_out/cost_time.jsonl gpurun_out/cost_ncu.jsonl MEASURED_PEAKS.json > gpurun_out/cost_tables.md; echo report_rc=$?
cat gpurun_out/cost_tables.md | head -24
