for rep in 1 2; do
for L in ${LIBS:-build/lib_*.so}; do
  NLSE_LIB=$PWD/$L timeout 300 python scripts/sweep.py 2>&1 | tail -1
done
done
