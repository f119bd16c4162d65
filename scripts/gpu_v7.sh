# carried-sum form (variant 7 = the new default, 12 transfers): parity subset + A/B timing
mkdir -p gpurun_out
PARITY_LOG=$PWD/gpurun_out/v7_parity.jsonl timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharding.py tests/test_abi.py -q -m gpu \
  -k "rk4_parity or constant or C4_core_box or 1d_stream_kernel_parity or lean_steps_bit or boundary_values or C2_full or C1_full or loopback_bitwise or fused_exchange_bitwise or caller_owned or padded_layout or msd" \
  > gpurun_out/v7_tests.log 2>&1; echo tests_rc=$?; tail -5 gpurun_out/v7_tests.log
AB_REPS=5 timeout 900 python scripts/ab_options.py C4:c64 C5W:c128 C3:c128 C2:c128 C2:c64 -- variant=5 variant=7 \
  > gpurun_out/ab_variant7.jsonl 2> gpurun_out/ab_variant7.err; echo ab_rc=$?; cut -c1-220 gpurun_out/ab_variant7.jsonl
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/v7_bench.json 2> gpurun_out/v7_bench.err; cut -c1-400 gpurun_out/v7_bench.json
