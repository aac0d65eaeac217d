#!/usr/bin/env bash
# Round-2 GPU session: microbenchmarks, GPU tests, smoke, bench (both arms), ncu launch list
# and one full capture of K1 / K2.  usage (under gpurun): bash tools/gpu_r2.sh <tag> [quick]
set -u
TAG=${1:-r2}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > "$OUT/nvsmi.txt" 2>&1
nproc > "$OUT/nproc.txt"
if [ -x tools/ubench ] && [ -n "${UBENCH:-}" ]; then timeout 120 tools/ubench > "$OUT/ubench.txt" 2>&1; fi
if [ -z "${NOTEST:-}" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest_gpu.log"
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?" >> "$OUT/smoke.log"
fi
timeout 900 python bench.py --steps 20 --warmup 3 > "$OUT/bench20.json" 2> "$OUT/bench20.err"
if [ -z "${QUICK:-}" ]; then
  timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > "$OUT/bench_ref.json" 2> "$OUT/bench_ref.err"
  timeout 900 python bench.py --headline-only --no-cpu-baseline > "$OUT/bench100.json" 2> "$OUT/bench100.err"
fi
if [ -n "${NCU:-}" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$OUT/launches.csv" \
      python bench.py --steps 4 --warmup 3 --no-cpu-baseline --headline-only > "$OUT/ncu_bench.log" 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_(compress|decompress)|k[12]x' -s 8 -c 2 \
      -o "$OUT/prof" -f python bench.py --steps 4 --warmup 3 --no-cpu-baseline --headline-only > "$OUT/ncu_full.log" 2>&1
  ncu -i "$OUT/prof.ncu-rep" --page raw --csv > "$OUT/raw.csv" 2>/dev/null
fi
echo done > "$OUT/DONE"
