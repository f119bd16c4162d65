mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharding.py -q -m gpu -k "lean or zchunk or path_options or V_array or loopback or nccl" > gpurun_out/c2_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/c2_tests.log
AB_REPS=3 timeout 600 python scripts/ab_options.py C4:c64 C5W:c64 C5W:c128 C3:c128 -- tile_schedule=0 tile_schedule=1 > gpurun_out/ab_sched.jsonl 2>&1; echo ab_rc=$?; cat gpurun_out/ab_sched.jsonl
for s in 0 1; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launch_sched$s.csv python scripts/one_step.py C4 c64 2 tile_schedule=$s > gpurun_out/ncu_sched$s.log 2>&1; echo ncu$s=$?
  python scripts/launches.py gpurun_out/launch_sched$s.csv 452984832
done
PROXY_STEPS=20 timeout 900 python scripts/loopback_proxy.py > gpurun_out/loopback_proxy.jsonl 2>&1; echo proxy_rc=$?; cat gpurun_out/loopback_proxy.jsonl
