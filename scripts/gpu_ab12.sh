for rep in 1 2; do
for lib in paper_1109_1027_b200/libnlse2shoc.so build/lib_rpw4.so; do
  NLSE_LIB=$lib timeout 120 python scripts/sweep_cfg.py C4 c64 20 2>&1 | tail -1
done
done
for lib in paper_1109_1027_b200/libnlse2shoc.so build/lib_rpw4.so; do
NLSE_LIB=$lib timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:stage_stream --csv --log-file gpurun_out/l_$(basename $lib).csv python scripts/sweep_cfg.py C4 c64 2 > /dev/null 2>&1
python scripts/launches.py gpurun_out/l_$(basename $lib).csv
done
