# A/B of compile variants on the cfg5 trilinear insert (620 frames in a 19 GB slab; wall ms per call)
for rep in 1 2; do
for L in default abtmp/*.so; do
  if [ "$L" = default ]; then unset SVR_LIB_PATH; else export SVR_LIB_PATH=$PWD/$L; fi
  echo "$L $(timeout 300 python tools/profile_config.py cfg5mid 4 2>/dev/null | grep 'insert wall' | tail -2 | tr '\n' ' ')"
done
done
