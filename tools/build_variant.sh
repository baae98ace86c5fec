#!/bin/bash
# tools/build_variant.sh <name> <nvcc -D flags...>: mla.cu rebuilt with the flags and linked with
# the in-tree objects of every other source into _variants/<name>.so (an A/B build, not shipped)
set -e
cd "$(dirname "$0")/.."
name=$1; shift
ARCH="-gencode arch=compute_100a,code=sm_100a"
mkdir -p _variants/obj
nvcc $ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr "$@" \
  -c paper_2605_05696_b200/csrc/mla.cu -o _variants/obj/mla_$name.o 2> _variants/obj/mla_$name.ptxas.txt
O=paper_2605_05696_b200/_lib/obj
nvcc $ARCH -shared -o _variants/$name.so $O/runtime.o $O/cdc.o $O/store.o $O/rotate.o $O/fanout.o \
  _variants/obj/mla_$name.o $O/prefix.o $O/ingest.o $O/exchange.o -lcuda -lpthread
grep -A2 "mla_reattach_2sm_v3" _variants/obj/mla_$name.ptxas.txt | grep -o "Used [0-9]* registers\|[0-9]* bytes spill stores" | tr '\n' ' '; echo " -> _variants/$name.so"
