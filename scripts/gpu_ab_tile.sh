# A/B of 3D complex64 tile shapes (alternating processes), plus a parity subset on the candidate
mkdir -p gpurun_out
NLSE_LIB=$PWD/ab/t128x12.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "rk4_parity_10_steps or tile_edge or lean_steps_bit or boundary_values" > gpurun_out/ab_tile_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/ab_tile_tests.log
LIBS="paper_1109_1027_b200/libnlse2shoc.so ab/t128x12.so" CFG="C4 c64" ROUNDS=3 AB_REPS=3 bash scripts/ab_libs.sh > gpurun_out/ab_tile_C4.jsonl 2>&1; cut -c1-260 gpurun_out/ab_tile_C4.jsonl
LIBS="paper_1109_1027_b200/libnlse2shoc.so ab/t128x12.so" CFG="C5W c64" ROUNDS=2 AB_REPS=3 bash scripts/ab_libs.sh > gpurun_out/ab_tile_C5W.jsonl 2>&1; cut -c1-260 gpurun_out/ab_tile_C5W.jsonl
NLSE_LIB=$PWD/ab/t128x12.so timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_C4_t128x12.csv python scripts/one_step.py C4 c64 2 > /dev/null 2>&1; echo ncu_rc=$?
python scripts/launches.py gpurun_out/launches_C4_t128x12.csv 452984832
