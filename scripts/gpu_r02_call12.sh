timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "1d or C2 or msd or fig1" > gpurun_out/c12_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/c12_tests.log
AB_REPS=5 timeout 600 python scripts/ab_options.py C2:c64 -- line_pairs=0 line_pairs=1 > gpurun_out/ab_c12.jsonl 2>&1; cat gpurun_out/ab_c12.jsonl
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launch_c2.csv python scripts/one_step.py C2 c64 2 > /dev/null 2>&1; echo ncu=$?
python scripts/launches.py gpurun_out/launch_c2.csv 4194304
