timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 120 -x > gpurun_out/gpu_all.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/gpu_all.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
python -c "import json;d=json.load(open('gpurun_out/bench.json'));print(d['value'], d['roofline'], d['clocks'], d.get('cpu_baseline'))"
timeout 900 python scripts/perf_table.py > gpurun_out/perf_table.jsonl 2>&1; echo perf_rc=$?; cat gpurun_out/perf_table.jsonl
