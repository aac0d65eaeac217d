#!/usr/bin/env bash
# Round-2 A/B: kbench of K1/K2 for each lib suffix in $LIBS at configs[1] and configs[3]
# sizes, K3 sweep, and the collective bench at TP=1 (peer leg).  usage: bash tools/gpu_ab2.sh <tag>
set -u
TAG=${1:-ab2}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
for rep in 1 2; do
for lib in ${LIBS:-default}; do
  if [ "$lib" = default ]; then L=paper_2604_24088_b200/libtaco_b200.so; else L=paper_2604_24088_b200/libtaco_b200_$lib.so; fi
  for N in ${NS:-20971520 83886080}; do
    echo -n "$lib " >> "$OUT/kbench.txt"
    TACO_B200_LIB=$L N=$N timeout 120 python tools/kbench.py 2>&1 | tr '\n' ' ' >> "$OUT/kbench.txt"; echo >> "$OUT/kbench.txt"
  done
  if [ -n "${K3:-}" ]; then echo "$lib" >> "$OUT/k3.txt"; TACO_B200_LIB=$L timeout 120 python tools/k3bench.py >> "$OUT/k3.txt" 2>&1; fi
done
done
if [ -n "${COLL:-}" ]; then timeout 600 python bench.py --collective --steps 20 --warmup 3 --no-cpu-baseline --size-sweep "" > "$OUT/bench_coll.json" 2> "$OUT/bench_coll.err"; fi
if [ -n "${TESTS:-}" ]; then timeout 900 python -m pytest $TESTS -q > "$OUT/pytest.log" 2>&1; echo rc=$? >> "$OUT/pytest.log"; fi
echo done > "$OUT/DONE"
