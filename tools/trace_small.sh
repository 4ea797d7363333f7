# CTA/tile timelines of small problems (ELSA_TRACE build in build/libelsa_trace.so)
export ELSA_LIB_PATH=$PWD/build/libelsa_trace.so
for sp in 1 8; do SHAPE=1,1,1024 SPLITS=$sp python tools/trace_ctas.py; done
SHAPE=8,12,512 SPLITS=0 python tools/trace_ctas.py
SHAPE=1,16,1024 SPLITS=1 python tools/trace_ctas.py
