# K5 A/B: in-tree build vs build/libelsa_<tag>.so (tools/time_tc.py, d = 64 and 128)
for t in base "$@"; do
  for D in 64 128; do
    if [ "$t" = base ]; then D=$D python tools/time_tc.py | sed "s/^/base /"
    else ELSA_LIB_PATH=$PWD/build/libelsa_$t.so D=$D python tools/time_tc.py | sed "s/^/$t /"; fi
  done
done
