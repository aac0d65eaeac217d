#!/usr/bin/env bash
# TC K1 A/B: correctness (TACO_B200_KERNELS=tc) + kbench of the default lib and each variant in $LIBS
set -u
OUT=gpurun_out/${1:-tcab}; mkdir -p $OUT
export TACO_B200_KERNELS=tc
timeout 300 python tools/tc_debug.py 148 300 640 > $OUT/tcdbg.log 2>&1
timeout 300 python -m pytest tests/test_gpu_codec.py -q -x -k "bf16_b256_k1_parity or config_size" > $OUT/pytest_tc.log 2>&1; echo rc=$? >> $OUT/pytest_tc.log
for lib in default ${LIBS:-}; do
  if [ "$lib" = default ]; then L=paper_2604_24088_b200/libtaco_b200.so; else L=paper_2604_24088_b200/libtaco_b200_$lib.so; fi
  echo -n "$lib " >> $OUT/kbench.txt; TACO_B200_LIB=$L B=256 timeout 120 python tools/kbench.py >> $OUT/kbench.txt 2>&1
done
TACO_B200_LIB=paper_2604_24088_b200/libtaco_b200_${NCU_LIB:-g1}.so timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_compress_tc" -s 3 -c 1 -o $OUT/prof -f python tools/kbench.py > $OUT/ncu.log 2>&1
echo done > $OUT/DONE
