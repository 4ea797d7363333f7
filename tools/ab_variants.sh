# A/B of compile variants in build/libelsa_<tag>.so against the in-tree build,
# alternating on one box: bash tools/ab_variants.sh tag1 tag2 ...
export AB_SHAPES=${AB_SHAPES:-1x16x16384,1x16x4096,8x12x512}
for i in 1 2; do
  python tools/ab_time.py base
  for t in "$@"; do ELSA_LIB_PATH=$PWD/build/libelsa_$t.so python tools/ab_time.py $t; done
done
