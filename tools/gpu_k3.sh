#!/usr/bin/env bash
# K3 iteration: collective/reduce GPU tests, collective bench line, launch list of the collective step
set -u
TAG=${1:-k3}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 900 python -m pytest tests -m gpu -q -x ${PYTEST_ARGS:--k "reduce or collective or allreduce"} > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest_gpu.log"
timeout 300 python bench.py --collective --cpu-seconds 1 > "$OUT/bench_coll.json" 2> "$OUT/bench_coll.err"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file "$OUT/launches_coll.csv" \
    python bench.py --collective --eager --steps 2 --warmup 1 --no-cpu-baseline > "$OUT/ncu_coll.log" 2>&1
echo done > "$OUT/DONE"
