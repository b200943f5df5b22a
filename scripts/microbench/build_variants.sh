#!/bin/bash
# Build libfractalsort variants with different k_scatter geometry (macros in wide.cu)
# into scripts/microbench/variants/<name>.so.  Usage: build_variants.sh name:"-DFOO=1 ..." ...
set -e
cd "$(dirname "$0")/../.."
ARCH="-gencode arch=compute_100a,code=sm_100a"
SRCS="abi hist16 scan expand16 wide partition host_stream trie peer small16"
mkdir -p scripts/microbench/variants
for spec in "$@"; do
  name="${spec%%:*}"; defs="${spec#*:}"
  d=build/var_$name; mkdir -p $d
  for f in $SRCS; do
    nvcc $ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude $defs -dc -o $d/$f.o paper_2605_10390_b200/csrc/$f.cu &
  done
  wait
  nvcc $ARCH -shared -Xcompiler -fPIC -o scripts/microbench/variants/$name.so $d/*.o
  echo built $name
done
