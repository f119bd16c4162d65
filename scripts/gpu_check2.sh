for a in "2 1030,9 c64" "2 530,9 c128" "3 100,100,12 c128" "3 200,100,12 c64"; do NLSE_LIB=$PWD/build/lib_dbg.so timeout 20 python scripts/lean_debug.py $a 2>&1 | sort | uniq -c | tail -2; done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharding.py -q -m gpu --timeout 120 -x > gpurun_out/gpu_all.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/gpu_all.log
