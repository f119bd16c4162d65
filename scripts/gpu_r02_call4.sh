mkdir -p gpurun_out
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_plain.log 2>&1; echo plain_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1; echo ncu_list_rc=$?
python scripts/launches.py gpurun_out/launches_bench.csv 452984832
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:stage_stream_kernel --launch-skip 4 --launch-count 4 -o gpurun_out/c4_step_full -f python scripts/one_step.py C4 c64 2 > gpurun_out/ncu_full.log 2>&1; echo ncu_full_rc=$?
timeout 2400 python scripts/c4_full_parity.py > gpurun_out/c4_full_parity.log 2>&1; echo c4full_rc=$?; tail -2 gpurun_out/c4_full_parity.log
