# round-2 final measurement set (under gpurun); outputs in gpurun_out/
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/smoke.log
rm -f gpurun_out/parity_final.jsonl
PARITY_LOG=$PWD/gpurun_out/parity_final.jsonl timeout 1500 python -m pytest tests -q -m gpu --durations=12 > gpurun_out/final_tests.log 2>&1; echo tests_rc=$?; tail -16 gpurun_out/final_tests.log
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo bench_rc=$?; cat gpurun_out/final_bench.json
timeout 300 python bench.py > gpurun_out/final_bench_default_flags.json 2> gpurun_out/final_bench_default_flags.err; echo bench_default_rc=$?
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/final_bench_torchrun1.json 2> gpurun_out/final_bench_torchrun1.err; echo torchrun1_rc=$?; tail -1 gpurun_out/final_bench_torchrun1.json | cut -c1-200
for wl in C5W C5S C3 C2; do
  timeout 600 python bench.py --steps 20 --warmup 5 --workload $wl --no-cpu-baseline > gpurun_out/final_bench_$wl.json 2> gpurun_out/final_bench_$wl.err; tail -1 gpurun_out/final_bench_$wl.json | cut -c1-200
done
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/final_bench_reference.json 2>&1; tail -1 gpurun_out/final_bench_reference.json | cut -c1-200
timeout 900 python scripts/perf_table.py > gpurun_out/final_perf_table.jsonl 2>&1; echo perf_rc=$?; cut -c1-200 gpurun_out/final_perf_table.jsonl
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/final_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu_list_rc=$?
python scripts/launches.py gpurun_out/final_launches.csv 452984832 | tee gpurun_out/final_launch_summary.txt
# NVTX ranges: only the kernels launched inside "nlse2shoc stage 1" ranges (expect the stage-1 mode only)
timeout 600 ncu --nvtx --nvtx-include "nlse2shoc stage 1/" --metrics gpu__time_duration.sum --clock-control none -c 20 --csv --log-file gpurun_out/final_nvtx_stage1.csv python scripts/one_step.py C5W c64 2 > /dev/null 2>&1; echo nvtx_rc=$?; grep -c stage_stream gpurun_out/final_nvtx_stage1.csv
# the full report is ~55 MB: keep it outside gpurun_out/ (64 MiB copy-back limit), bring back
# the summary and the per-instruction source page
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:stage_stream_kernel --launch-skip 4 --launch-count 4 -o /tmp/final_step_full -f python scripts/one_step.py C4 c64 2 > /dev/null 2>&1; echo ncu_full_rc=$?
python scripts/ncu_summary.py /tmp/final_step_full.ncu-rep > gpurun_out/final_stage_summary.txt; head -16 gpurun_out/final_stage_summary.txt
ncu -i /tmp/final_step_full.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/final_stage_source.csv.gz
