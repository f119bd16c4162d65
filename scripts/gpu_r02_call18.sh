AB_REPS=3 timeout 900 python scripts/ab_options.py C4:c64 C3:c128 -- variant=1 variant=3 > gpurun_out/ab_c18.jsonl 2>&1; cut -c1-125 gpurun_out/ab_c18.jsonl
