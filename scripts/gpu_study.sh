# study captures: --set full of one step's four stage launches (C5W c128 and C4 c64), with stall
# samples per SASS instruction of the stages of interest
mkdir -p gpurun_out
for cfg in "C5W c128" "C4 c64"; do
  set -- $cfg
  tag=$1_$2
  timeout 1200 ncu --set full --import-source on --clock-control none -k regex:stage_stream_kernel --launch-skip 4 --launch-count 4 -o /tmp/study_$tag -f python scripts/one_step.py $1 $2 2 > /dev/null 2>&1; echo ncu_$tag rc=$?
  python scripts/ncu_summary.py /tmp/study_$tag.ncu-rep > gpurun_out/study_${tag}_summary.txt
  ncu -i /tmp/study_$tag.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/study_${tag}_source.csv.gz
done
head -70 gpurun_out/study_C5W_c128_summary.txt
