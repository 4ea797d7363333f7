#!/bin/bash
# Time every build/var_*.so with each forced forward config on AB_SHAPES
# (default 4K and 16K); CFGS overrides the config list.
for v in build/var_*.so; do
  n=$(basename $v .so)
  for c in ${CFGS:-w8r16 w8r8 w4r8}; do
    AB_SHAPES=${AB_SHAPES:-1x16x4096,1x16x16384} ELSA_FWD_CFG=$c ELSA_LIB_PATH=$v timeout 150 python tools/ab_time.py ${n}_$c || echo "$v $c failed"
  done
done
