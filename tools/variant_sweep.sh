#!/bin/bash
# Build libelsa variants (compile-time knobs of fwd_f32.cuh / ptxas options)
# into build/var_<name>.so:  tools/variant_sweep.sh "name:flags" ...
# Time them on a GPU box with:
#   for v in build/var_*.so; do ELSA_LIB_PATH=$v python tools/ab_time.py $(basename $v .so); done
set -e
cd "$(dirname "$0")/.."
mkdir -p build
ARCH="-gencode arch=compute_100a,code=sm_100a"
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  [ "$name" = "$spec" ] && flags=""
  nvcc $ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -Iinclude \
       -Ipaper_2604_23798_b200/csrc $flags -o build/var_$name.so \
       paper_2604_23798_b200/csrc/elsa_abi.cu &
done
wait
ls build/var_*.so
