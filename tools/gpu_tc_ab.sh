#!/usr/bin/env bash
# TC K1 A/B: correctness + kbench of the default lib and each variant in $LIBS, one ncu capture
set -u
OUT=gpurun_out/${1:-tcab}; mkdir -p $OUT
timeout 300 python tools/tc_debug.py 148 300 640 > $OUT/tcdbg.log 2>&1
timeout 300 python -m pytest tests/test_gpu_codec.py -q -x -k "tensor_core or config_size" > $OUT/pytest_tc.log 2>&1; echo rc=$? >> $OUT/pytest_tc.log
for lib in default ${LIBS:-}; do
  if [ "$lib" = default ]; then L=paper_2604_24088_b200/libtaco_b200.so; else L=paper_2604_24088_b200/libtaco_b200_$lib.so; fi
  echo -n "$lib " >> $OUT/kbench.txt; TACO_B200_LIB=$L B=256 timeout 120 python tools/kbench.py >> $OUT/kbench.txt 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_compress_tc" -s 3 -c 1 -o $OUT/prof -f python tools/kbench.py > $OUT/ncu.log 2>&1
echo done > $OUT/DONE
