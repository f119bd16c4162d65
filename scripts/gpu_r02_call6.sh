LIBS="ab/lib_dyn_nofused.so paper_1109_1027_b200/libnlse2shoc.so" CFG="C4 c64" ROUNDS=3 bash scripts/ab_libs.sh > gpurun_out/ab_libs_c6.jsonl 2>&1; cat gpurun_out/ab_libs_c6.jsonl
PROXY_STEPS=20 timeout 900 python scripts/loopback_proxy.py > gpurun_out/loopback_proxy_fused2.jsonl 2>&1; cat gpurun_out/loopback_proxy_fused2.jsonl
