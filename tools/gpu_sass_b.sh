#!/usr/bin/env bash
# source-level ncu capture of K1 / K2 at block size $B via kbench, + SASS histograms
set -u
OUT=gpurun_out/${1:-sassb}
mkdir -p "$OUT"
B=${B:-64} REPS=3 timeout 900 ncu --set full --import-source on --clock-control none -k regex:'k_(compress|decompress)' -s 12 -c 2 \
    -o "$OUT/prof" -f python tools/kbench.py > "$OUT/ncu_full.log" 2>&1
for id in 0 1; do
  ncu -i "$OUT/prof.ncu-rep" --page source --csv --print-source sass --launch-skip $id --launch-count 1 > "$OUT/src_$id.csv" 2>/dev/null
  python tools/sass_hist.py "$OUT/src_$id.csv" 30 > "$OUT/hist_$id.txt" 2>&1
done
ncu -i "$OUT/prof.ncu-rep" --page raw --csv > "$OUT/raw.csv" 2>/dev/null
echo done > "$OUT/DONE"
