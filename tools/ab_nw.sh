# A/B of libdmb200 variants (tools/build_variant.sh) on the NW throughput kernel
for v in base u2 u4 base u2 u4; do
  if [ $v = base ]; then L=; else L=_variants/$v/libdmb200.so; fi
  echo "$v $(DM_LIB_PATH=$L python tools/prof_nw.py --pairs 65536 --len 1000 --reps 3 2>&1 | tail -1)"
done
