AB_REPS=3 timeout 900 python scripts/ab_options.py C4:c64 C5W:c64 C5W:c128 -- zchunks=0 zchunks=6 zchunks=4 zchunks=3 zchunks=24 > gpurun_out/ab_zchunks.jsonl 2>&1; cat gpurun_out/ab_zchunks.jsonl
