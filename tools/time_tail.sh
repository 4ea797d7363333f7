# Tail split A/B: ELSA_TAIL=0 (off), 1 (cost model), s (force s pieces) on the
# shapes whose last wave is partly empty; CUDA-graph replays, L2 flushed.
export AB_SHAPES=8x12x512,4x12x512,8x16x512,1x16x4096,2x16x2048
for t in 0 1 2 3 4 6 8; do
  ELSA_TAIL=$t python tools/ab_time.py tail$t
done
