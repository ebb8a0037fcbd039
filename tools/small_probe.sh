# kernel durations (ncu) of encode + decode at small chunk sizes, per variants/* build (dev tool)
for d in variants/*/; do
  for e in 32768 524288 2097152; do
    echo "== $d $e"
    FC2_LIB=$d/libfc2.so ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_encode|k_decode" -s 4 -c 2 python tools/prof_codec.py --elems $e --reps 4 2>&1 | grep -E "^  void|duration" | sed 's/(fc2::.*//; s/ *gpu__time_duration.sum *us */ /'
  done
done
