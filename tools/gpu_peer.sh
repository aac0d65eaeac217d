#!/usr/bin/env bash
# peer-memory collective iteration: peer tests, codec/collective regression, timings
set -u
TAG=${1:-peer}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 900 python -m pytest tests/test_gpu_peer.py -q -x > "$OUT/pytest_peer.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest_peer.log"
if [ -z "${QUICK:-}" ]; then
  timeout 900 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_peer.py > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest_gpu.log"
fi
timeout 300 python tools/peer_prof.py > "$OUT/peer_prof.txt" 2>&1
ITERS=3 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file "$OUT/launches_peer.csv" python tools/peer_prof.py > "$OUT/ncu_peer.log" 2>&1
timeout 300 python bench.py --collective --cpu-seconds 1 > "$OUT/bench_coll.json" 2> "$OUT/bench_coll.err"
echo done > "$OUT/DONE"
