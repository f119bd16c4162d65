#!/bin/bash
# A/B timing of library builds and env settings (scripts/sweep_cfg.py: best-of-3 x K steps,
# CUDA events).  Every JSON line is prefixed with its label.  Examples:
#   LIBS="paper_1109_1027_b200/libnlse2shoc.so build/lib_x.so" CFGS="C4:c64 C5W:c128" bash scripts/ab.sh
#   ENVS="NLSE_TMA_PROMO=0 NLSE_TMA_PROMO=64" CFGS="C4:c64" REPS=3 bash scripts/ab.sh
LIBS=${LIBS:-paper_1109_1027_b200/libnlse2shoc.so}
ENVS=${ENVS:-NONE=0}
CFGS=${CFGS:-C4:c64}
REPS=${REPS:-2}
K=${K:-20}
for rep in $(seq $REPS); do
  for lib in $LIBS; do
    for e in $ENVS; do
      for c in $CFGS; do
        env NLSE_LIB=$lib $e timeout 120 python scripts/sweep_cfg.py ${c%%:*} ${c##*:} $K 2>&1 | tail -1 \
          | sed "s|^|$(basename $lib) $e |"
      done
    done
  done
done
