#!/usr/bin/env bash
# Build A/B variants of libtaco_b200.so with extra nvcc defines (kept out of the package
# dir's default name): tools/build_variants.sh name "-DFOO=1" [name2 "-D..."] ...
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  make -s -j8 -C "$ROOT/paper_2604_24088_b200/csrc" BUILD="$ROOT/paper_2604_24088_b200/csrc/_build_$name" \
       LIB="$ROOT/paper_2604_24088_b200/libtaco_b200_$name.so" NVEXTRA="$flags" &
done
wait
