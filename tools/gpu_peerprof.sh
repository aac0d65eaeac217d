#!/usr/bin/env bash
set -u
OUT=gpurun_out/${1:-pp}
mkdir -p "$OUT"
timeout 300 python tools/peer_prof.py > "$OUT/peer_prof.txt" 2>&1
ITERS=3 REPS=3 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file "$OUT/launches_peer.csv" python tools/peer_prof.py > "$OUT/ncu_peer.log" 2>&1
echo done > "$OUT/DONE"
