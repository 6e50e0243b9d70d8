#!/bin/bash
# Build libisq variants (compile-time tunables) next to the main library:
#   bash tools/build_variants.sh name1 "-DFLAG=.." name2 "-DFLAG=.." ...
# -> build/variants/<name>/libisq.so, selected at run time with ISQ_LIBRARY=...
set -e
cd "$(dirname "$0")/.."
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  mkdir -p build/variants/$name
  ISQ_NVCC_EXTRA="$flags" ISQ_BUILD_DIR=build/variants/$name/obj ISQ_LIBRARY=build/variants/$name/libisq.so \
    python paper_1809_11134_b200/_build.py --force > build/variants/$name/build.log 2>&1 || { cat build/variants/$name/build.log; exit 1; }
  cp build/variants/$name/obj/ptxas.log build/variants/$name/ptxas.log; rm -rf build/variants/$name/obj
  echo "built $name ($flags)"
done
