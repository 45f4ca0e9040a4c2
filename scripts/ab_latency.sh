for n in base new base new; do
  if [ $n = base ]; then export RTN_LIB=$PWD/build_var/lib_base.so; else unset RTN_LIB; fi
  echo "== $n"
  timeout 100 python scripts/decomp_probe.py c3 1x1
  timeout 100 python scripts/decomp_probe.py c1 1x1
done
