#!/bin/bash
# Build libfractalsort variants with different compile-time macros into
# scripts/microbench/variants/<name>.so.  Usage: build_variants.sh name:"-DFOO=1 ..." ...
# VARSRC="hist16 expand16" rebuilds only those sources with the macros and links
# the other objects from build/ (run `make` first); default: every source.
set -e
cd "$(dirname "$0")/../.."
ARCH="-gencode arch=compute_100a,code=sm_100a"
ALL="abi hist16 scan expand16 wide partition host_stream trie peer small16 exchange nvls"
SRCS="${VARSRC:-$ALL}"
mkdir -p scripts/microbench/variants
for spec in "$@"; do
  name="${spec%%:*}"; defs="${spec#*:}"
  d=build/var_$name; rm -rf $d; mkdir -p $d
  for f in $ALL; do
    if [[ " $SRCS " == *" $f "* ]]; then
      nvcc $ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude $defs -dc -o $d/$f.o paper_2605_10390_b200/csrc/$f.cu &
    else
      cp build/$f.o $d/$f.o
    fi
  done
  wait
  for f in $SRCS; do [ -f $d/$f.o ] || { echo "variant $name: $f.cu failed to compile" >&2; exit 1; }; done
  nvcc $ARCH -shared -Xcompiler -fPIC -o scripts/microbench/variants/$name.so $d/*.o
  echo built $name
done
