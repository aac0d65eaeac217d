#!/usr/bin/env bash
# One gpurun session: GPU tests, smoke, bench (both arms), ncu launch list + one full capture.
# usage (under gpurun): bash tools/gpu_round.sh [tag]
set -u
TAG=${1:-r1}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > "$OUT/nvsmi.txt" 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest_gpu.log"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?" >> "$OUT/smoke.log"
timeout 600 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > "$OUT/bench_ref.json" 2> "$OUT/bench_ref.err"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$OUT/launches.csv" \
    python bench.py --steps 4 --warmup 3 --no-cpu-baseline > "$OUT/ncu_bench.log" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_(compress|decompress)' -s 6 -c 2 \
    -o "$OUT/prof" -f python bench.py --steps 4 --warmup 3 --no-cpu-baseline > "$OUT/ncu_full.log" 2>&1
ncu -i "$OUT/prof.ncu-rep" --page raw --csv > "$OUT/raw.csv" 2>/dev/null
ncu -i "$OUT/prof.ncu-rep" --page details --csv > "$OUT/ncu_details.csv" 2>/dev/null
python tools/ncu_summary.py "$OUT/raw.csv" "$TAG" "$OUT/${TAG}_ncu_traffic.json" > /dev/null 2>&1
timeout 300 python bench.py --collective > "$OUT/bench_coll.json" 2> "$OUT/bench_coll.err"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file "$OUT/launches_coll.csv" \
    python bench.py --collective --eager --steps 2 --warmup 1 --no-cpu-baseline > "$OUT/ncu_coll.log" 2>&1
bash tools/gpu_reftests.sh "$TAG/reftests" > /dev/null 2>&1
echo done > "$OUT/DONE"
