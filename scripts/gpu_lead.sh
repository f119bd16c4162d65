for rep in 1 2; do
for LD in 0 2 4 8; do
  echo "pairlead=$LD $(NLSE_LEAD=$LD NLSE_LEAD_PAIR=1 timeout 120 python scripts/sweep.py 2>&1 | tail -1)"
done
done
NLSE_LEAD=4 NLSE_LEAD_PAIR=1 timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
NLSE_LEAD=4 NLSE_LEAD_PAIR=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_pl.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu_rc=$?
