# A/B of the per-tile W accumulator (ELSA_TILE_ACC) on one box; build/libelsa_acc0.so
# is the same source with -DELSA_TILE_ACC=0
export AB_SHAPES=1x16x1024,1x16x4096,1x16x8192,1x16x16384,8x12x512,1x1x1024
for i in 1 2; do
  ELSA_LIB_PATH=$PWD/build/libelsa_acc0.so python tools/ab_time.py acc0 >> gpurun_out/ab_acc.txt 2>&1
  python tools/ab_time.py acc >> gpurun_out/ab_acc.txt 2>&1
done
python tools/chain_error.py > gpurun_out/chain_acc.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gputest2.log 2>&1
