# A/B: build/libelsa_prev.so (previous commit) vs the in-tree build, alternating
export AB_SHAPES=${AB_SHAPES:-1x16x16384,1x16x8192,1x16x4096,8x12x512}
for i in 1 2; do
  ELSA_LIB_PATH=$PWD/build/libelsa_prev.so python tools/ab_time.py prev
  python tools/ab_time.py cur
done
