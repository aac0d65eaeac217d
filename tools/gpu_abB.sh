#!/usr/bin/env bash
# K1/K2 A/B over block sizes at the configs[2] per-rank size (libs in $LIBS), then parity tests
OUT=gpurun_out/${1:-abB}; mkdir -p $OUT
for rep in 1 2; do for lib in ${LIBS:-default}; do
  if [ $lib = default ]; then L=paper_2604_24088_b200/libtaco_b200.so; else L=paper_2604_24088_b200/libtaco_b200_$lib.so; fi
  for B in ${BS:-64 256}; do
    echo -n "$lib " >> $OUT/k.txt; TACO_B200_LIB=$L B=$B N=58720256 timeout 120 python tools/kbench.py 2>&1 | tr "\n" " " >> $OUT/k.txt; echo >> $OUT/k.txt
  done
done; done
if [ -n "${TESTS:-}" ]; then timeout 900 python -m pytest $TESTS -q > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log; fi
