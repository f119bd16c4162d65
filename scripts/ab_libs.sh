# Alternating A/B of library builds on one config (each run a fresh process; best of REPS x K steps):
#   LIBS="ab/a.so paper_1109_1027_b200/libnlse2shoc.so" CFG="C4 c64" ROUNDS=3 bash scripts/ab_libs.sh
ROUNDS=${ROUNDS:-3}
for r in $(seq $ROUNDS); do
  for L in $LIBS; do
    NLSE_LIB=$PWD/$L AB_REPS=${AB_REPS:-3} timeout 300 python scripts/ab_options.py ${CFG// /:} -- ${SETS:-tile_schedule=2} 2>&1 | grep "^{" | sed "s|^|{\"lib\": \"$L\", \"round\": $r, \"r\": |; s|\$|}|"
  done
done
