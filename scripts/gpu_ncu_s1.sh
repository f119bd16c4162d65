timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharding.py -q -m gpu --timeout 120 -x > gpurun_out/gpu_all.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/gpu_all.log
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stage_stream -s 12 -c 4 -o gpurun_out/prof_c4 -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu2.log 2>&1; echo ncu2_rc=$?
