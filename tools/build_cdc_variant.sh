#!/bin/bash
# tools/build_cdc_variant.sh <name> <nvcc -D flags...>: cdc.cu rebuilt with the flags and linked with
# the in-tree objects of every other source into _variants/<name>.so (an A/B build, not shipped)
set -e
cd "$(dirname "$0")/.."
name=$1; shift
ARCH="-gencode arch=compute_100a,code=sm_100a"
mkdir -p _variants/obj
nvcc $ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr "$@" \
  -c paper_2605_05696_b200/csrc/cdc.cu -o _variants/obj/cdc_$name.o 2> _variants/obj/cdc_$name.ptxas.txt
O=paper_2605_05696_b200/_lib/obj
nvcc $ARCH -shared -o _variants/$name.so $O/runtime.o _variants/obj/cdc_$name.o $O/store.o $O/rotate.o $O/fanout.o \
  $O/mla.o $O/prefix.o $O/ingest.o $O/exchange.o -lcuda -lpthread
echo " -> _variants/$name.so"
