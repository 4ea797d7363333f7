#!/bin/bash
# Bench the forward kernel under each ELSA_FWD_CFG (kernel-only sweep, no CPU baseline)
mkdir -p gpurun_out
for cfg in ${CFGS:-w4r8 w8r8 w8r16}; do
  ELSA_FWD_CFG=$cfg timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/cfg_$cfg.log 2>&1
done
echo done
