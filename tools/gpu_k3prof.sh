#!/usr/bin/env bash
# K3 (reduce-encode) profile at configs[1] TP=2: timing sweep, one ncu --set full capture with
# SASS source, raw metrics.  usage (under gpurun): bash tools/gpu_k3prof.sh <tag>
set -u
TAG=${1:-k3}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
PS="1 2 4 8" timeout 300 python tools/k3bench.py > "$OUT/k3.txt" 2>&1
PS="2" REPS=5 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k3x -s 3 -c 1 \
    -o "$OUT/prof" -f python tools/k3bench.py > "$OUT/ncu.log" 2>&1
ncu -i "$OUT/prof.ncu-rep" --page raw --csv > "$OUT/raw.csv" 2>/dev/null
ncu -i "$OUT/prof.ncu-rep" --page source --csv --print-source sass > "$OUT/src_k3x.csv" 2>/dev/null
ncu -i "$OUT/prof.ncu-rep" --page details --csv > "$OUT/details.csv" 2>/dev/null
rm -f "$OUT/prof.ncu-rep"
echo done > "$OUT/DONE"
