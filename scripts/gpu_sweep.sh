for L in build/lib_*.so; do
  NLSE_LIB=$PWD/$L timeout 300 python scripts/sweep.py 2>&1 | tail -1
done
NLSE_LIB=$PWD/build/lib_ty28w14r2.so timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
