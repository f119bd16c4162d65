for L in paper_1109_1027_b200/libnlse2shoc.so build/lib_cfg2.so; do
  NLSE_LIB=$PWD/$L timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_ab.log 2>&1; echo $L smoke_rc=$? $(tail -1 gpurun_out/smoke_ab.log)
  NLSE_LIB=$PWD/$L timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_ab.json 2>&1; echo $L $(python -c "import json;d=json.load(open('gpurun_out/bench_ab.json'));print(d['value'], d['roofline']['achieved'], d['clocks'])")
  NLSE_LIB=$PWD/$L timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_$(basename $L).csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
done
