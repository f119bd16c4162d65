AB_REPS=3 timeout 900 python scripts/ab_options.py C4:c64 -- zchunks=0 zchunks=12 loopback=8 loopback=8,zchunks=3 > gpurun_out/ab_c16a.jsonl 2>&1; cut -c1-125 gpurun_out/ab_c16a.jsonl
AB_REPS=3 timeout 900 python scripts/ab_options.py C5W:c64 C5W:c128 -- zchunks=0 zchunks=3 zchunks=4 zchunks=6 > gpurun_out/ab_c16b.jsonl 2>&1; cut -c1-125 gpurun_out/ab_c16b.jsonl
