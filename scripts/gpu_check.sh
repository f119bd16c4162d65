set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
tail -2 gpurun_out/smoke.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 600 -x > gpurun_out/gpu_all.log 2>&1; echo all_rc=$?
tail -40 gpurun_out/gpu_all.log
