# study captures: launch list and --set full of one step's four stage launches for a config
mkdir -p gpurun_out
# usage: bash scripts/gpu_study.sh ["CFG DTYPE NPOINTS" ...]
if [ $# -eq 0 ]; then set -- "C3 c128 67108864" "C2 c128 4194304"; fi
for cfg in "$@"; do
  set -- $cfg
  tag=$1_$2
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file gpurun_out/study_launches_$tag.csv python scripts/one_step.py $1 $2 2 > /dev/null 2>&1
  python scripts/launches.py gpurun_out/study_launches_$tag.csv $3
  timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"stage_stream_kernel|line_stream_kernel" --launch-skip 4 --launch-count 4 -o /tmp/study_$tag -f python scripts/one_step.py $1 $2 2 > /dev/null 2>&1; echo ncu_$tag rc=$?
  python scripts/ncu_summary.py /tmp/study_$tag.ncu-rep > gpurun_out/study_${tag}_summary.txt
  ncu -i /tmp/study_$tag.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/study_${tag}_source.csv.gz
done
