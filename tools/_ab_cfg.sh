# A/B of compile variants on one config's insert: tools/_ab_cfg.sh cfg3
for rep in 1 2 3; do
for L in default abtmp/*.so; do
  if [ "$L" = default ]; then unset SVR_LIB_PATH; else export SVR_LIB_PATH=$PWD/$L; fi
  echo "$L $(timeout 300 python tools/time_config.py $1 5 2>/dev/null | tail -1)"
done
done
