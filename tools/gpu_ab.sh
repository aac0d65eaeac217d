#!/usr/bin/env bash
# A/B of kernel variants: for every lib in $LIBS (suffixes; "" = default) and every family in
# $FAMS (r2 tile reg) run tools/kbench.py for each block size in $BS and dtype in $DTS.
set -u
TAG=${1:-ab}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
if [ -z "${NOTEST:-}" ]; then
  timeout 900 python -m pytest tests -m gpu -q -x ${PYTEST_ARGS:-} > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest_gpu.log"
fi
for lib in ${LIBS:-default}; do
  if [ "$lib" = default ]; then L=paper_2604_24088_b200/libtaco_b200.so; else L=paper_2604_24088_b200/libtaco_b200_$lib.so; fi
  for fam in ${FAMS:-r2}; do
    for B in ${BS:-256}; do
      for DT in ${DTS:-bf16}; do
        echo -n "$lib " >> "$OUT/kbench.txt"
        TACO_B200_LIB=$L TACO_B200_KERNELS=$fam DT=$DT B=$B timeout 120 python tools/kbench.py >> "$OUT/kbench.txt" 2>&1
      done
    done
  done
done
if [ -n "${BENCH:-}" ]; then timeout 600 python bench.py --cpu-seconds 2 > "$OUT/bench.json" 2> "$OUT/bench.err"; fi
if [ -n "${NCU:-}" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${NCU_K:-k_(compress|decompress)}" -s 6 -c 2 \
      -o "$OUT/prof" -f python bench.py --steps 4 --warmup 3 --no-cpu-baseline > "$OUT/ncu_full.log" 2>&1
fi
echo done > "$OUT/DONE"
