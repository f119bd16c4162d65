mkdir -p gpurun_out
NLSE_LIB=$PWD/ab/occ2.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "rk4_parity_10_steps or tile_edge or boundary_values or laplacian_parity" > gpurun_out/ab2d_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/ab2d_tests.log
LIBS="paper_1109_1027_b200/libnlse2shoc.so ab/occ2.so" CFG="C3 c128" ROUNDS=3 AB_REPS=3 bash scripts/ab_libs.sh > gpurun_out/ab_occ2_C3.jsonl 2>&1; cut -c1-260 gpurun_out/ab_occ2_C3.jsonl
NLSE_LIB=$PWD/ab/occ2.so timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_C3_occ2.csv python scripts/one_step.py C3 c128 2 > /dev/null 2>&1; echo ncu_rc=$?
python scripts/launches.py gpurun_out/launches_C3_occ2.csv 67108864
