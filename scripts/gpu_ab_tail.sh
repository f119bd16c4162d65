# TAIL_CHUNKS A/B (short end z-chunks) + its parity tests; outputs in gpurun_out/
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "tail or path_options or zchunk or tile_edge or C4_full or C3_full or C5W_full or loopback or cached" > gpurun_out/s3_tail_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/s3_tail_tests.log
AB_REPS=5 timeout 900 python scripts/ab_options.py C4:c64 C5W:c64 C5W:c128 C3:c128 C3:c64 -- tail_chunks=1 tail_chunks=0 tail_chunks=1 tail_chunks=0 > gpurun_out/s3_ab_tail.jsonl 2>&1; echo ab_rc=$?; cut -c1-160 gpurun_out/s3_ab_tail.jsonl
AB_REPS=4 timeout 900 python scripts/ab_options.py C4:c64 -- loopback=8,tail_chunks=1 loopback=8,tail_chunks=0 loopback=2,tail_chunks=1 loopback=2,tail_chunks=0 tail_chunks=1 > gpurun_out/s3_ab_tail_loop.jsonl 2>&1; echo ab2_rc=$?; cut -c1-160 gpurun_out/s3_ab_tail_loop.jsonl
