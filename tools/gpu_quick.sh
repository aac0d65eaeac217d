#!/usr/bin/env bash
# quick GPU iteration: gpu tests + kernel A/B (register vs tile kernels) + bench line
set -u
TAG=${1:-q}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 900 python -m pytest tests -m gpu -q -x ${PYTEST_ARGS:-} > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest_gpu.log"
for B in ${BS:-256}; do
  TACO_B200_KERNELS=reg B=$B timeout 120 python tools/kbench.py >> "$OUT/kbench.txt" 2>&1
  B=$B timeout 120 python tools/kbench.py >> "$OUT/kbench.txt" 2>&1
  DT=f32 B=$B timeout 120 python tools/kbench.py >> "$OUT/kbench.txt" 2>&1
done
timeout 600 python bench.py --cpu-seconds 2 > "$OUT/bench.json" 2> "$OUT/bench.err"
if [ -n "${NCU:-}" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_(compress|decompress)' -s 6 -c 2 \
      -o "$OUT/prof" -f python bench.py --steps 4 --warmup 3 --no-cpu-baseline > "$OUT/ncu_full.log" 2>&1
fi
echo done > "$OUT/DONE"
