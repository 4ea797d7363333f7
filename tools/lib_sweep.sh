#!/bin/bash
# Bench alternative library builds (ELSA_LIB_PATH) x configs (ELSA_FWD_CFG)
mkdir -p gpurun_out
for lib in ${LIBS:-libelsa.so}; do
  for cfg in ${CFGS:-w8r16}; do
    ELSA_LIB_PATH=$PWD/paper_2604_23798_b200/$lib ELSA_FWD_CFG=$cfg timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/lib_${lib%.so}_$cfg.log 2>&1
  done
done
echo done
