#!/usr/bin/env bash
# PDL A/B: tests with PDL on, kernel timings and the bench line with TACO_PDL=0/1
set -u
OUT=gpurun_out/${1:-pdl}
mkdir -p "$OUT"
timeout 900 python -m pytest tests -m gpu -q -x > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest_gpu.log"
for P in 0 1; do
  for N in 5242880 20971520 83886080; do
    for DT in bf16 f32; do
      echo -n "pdl=$P " >> "$OUT/kbench.txt"; TACO_PDL=$P N=$N DT=$DT B=256 timeout 120 python tools/kbench.py >> "$OUT/kbench.txt" 2>&1
    done
  done
  TACO_PDL=$P timeout 300 python bench.py --cpu-seconds 1 > "$OUT/bench_pdl$P.json" 2> "$OUT/bench_pdl$P.err"
  TACO_PDL=$P timeout 300 python bench.py --collective --no-cpu-baseline > "$OUT/bench_coll_pdl$P.json" 2> "$OUT/bench_coll_pdl$P.err"
done
echo done > "$OUT/DONE"
