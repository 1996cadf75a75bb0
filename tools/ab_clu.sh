for v in base notrace nowait; do
  if [ $v = base ]; then L=; else L=_variants/$v/libdmb200.so; fi
  echo "== $v"; DM_LIB_PATH=$L python tools/nw_latency.py --pairs 1 --len 2600 --reps 3 2>&1 | tail -4
done
