#!/usr/bin/env bash
# tensor-core K1 check: parity tests, kernel A/B (tc vs CUDA-core), one ncu capture per lib
set -u
OUT=gpurun_out/${1:-tc1}; mkdir -p $OUT
timeout 300 python -m pytest tests/test_gpu_codec.py -q -x -k "tensor_core or config_size" > $OUT/pytest_tc.log 2>&1; echo rc=$? >> $OUT/pytest_tc.log
for lib in ${LIBS:-default}; do
  if [ "$lib" = default ]; then L=paper_2604_24088_b200/libtaco_b200.so; else L=paper_2604_24088_b200/libtaco_b200_$lib.so; fi
  for fam in default cuda; do echo -n "$lib " >> $OUT/kbench.txt; TACO_B200_LIB=$L TACO_B200_KERNELS=$fam B=256 timeout 120 python tools/kbench.py >> $OUT/kbench.txt 2>&1; done
  TACO_B200_LIB=$L timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_compress_tc" -s 3 -c 1 -o $OUT/prof_$lib -f python tools/kbench.py > $OUT/ncu_$lib.log 2>&1
done
echo done > $OUT/DONE
