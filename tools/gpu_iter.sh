#!/usr/bin/env bash
# Kernel iteration loop (under gpurun): GPU tests, headline bench, one ncu --set full capture
# of K1 / K2 with SASS-level source.  usage: bash tools/gpu_iter.sh <tag>
set -u
TAG=${1:-iter}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
if [ -z "${NOTEST:-}" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest_gpu.log"
fi
timeout 600 python bench.py --steps 50 --warmup 5 --headline-only --no-cpu-baseline ${BENCH_ARGS:-} > "$OUT/bench.json" 2> "$OUT/bench.err"
if [ -z "${NONCU:-}" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${NCU_K:-k[123]x|k_}" -s 8 -c ${NCU_C:-2} \
      -o "$OUT/prof" -f python bench.py --steps 4 --warmup 3 --no-cpu-baseline --headline-only ${BENCH_ARGS:-} > "$OUT/ncu_full.log" 2>&1
  for k in k1x k2x k3x; do
    ncu -i "$OUT/prof.ncu-rep" --page source --csv --print-source sass -k regex:$k > "$OUT/src_$k.csv" 2>/dev/null
  done
  ncu -i "$OUT/prof.ncu-rep" --page raw --csv > "$OUT/raw.csv" 2>/dev/null
  rm -f "$OUT/prof.ncu-rep"
fi
echo done > "$OUT/DONE"
