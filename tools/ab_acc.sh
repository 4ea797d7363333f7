# A/B of the long-chain two-level-accumulator kernel (w8r8acc) against w8r8
# on one box (forced configurations), plus the chain-length error sweep
for i in 1 2; do
  for c in w8r8 w8r8acc; do
    ELSA_FWD_CFG=$c AB_SHAPES=1x16x4096,1x16x8192,1x16x16384 python tools/ab_time.py $c
  done
done
python tools/chain_error.py
