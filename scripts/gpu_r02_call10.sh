for cfg in "C4 c64" "C2 c64" "C2 c128" "C3 c128" "C5W c128"; do
LIBS="ab/lib_unroll3.so paper_1109_1027_b200/libnlse2shoc.so" CFG="$cfg" ROUNDS=2 bash scripts/ab_libs.sh
done > gpurun_out/ab_align.jsonl 2>&1; cat gpurun_out/ab_align.jsonl
LIBS="ab/lib_unroll3.so paper_1109_1027_b200/libnlse2shoc.so" CFG="C4 c64" SETS="variant=1 variant=3" ROUNDS=1 bash scripts/ab_libs.sh > gpurun_out/ab_align_two.jsonl 2>&1; cat gpurun_out/ab_align_two.jsonl
