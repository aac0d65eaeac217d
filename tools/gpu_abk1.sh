#!/usr/bin/env bash
# K1 A/B (lib suffixes in $LIBS) for bf16 and fp32 at configs[1] / configs[3] sizes, 2 reps
OUT=gpurun_out/${1:-abk1}; mkdir -p $OUT
for rep in 1 2; do for lib in ${LIBS:-default}; do
  if [ $lib = default ]; then L=paper_2604_24088_b200/libtaco_b200.so; else L=paper_2604_24088_b200/libtaco_b200_$lib.so; fi
  for DT in bf16 f32; do for N in 20971520 83886080; do
    echo -n "$lib " >> $OUT/k.txt; TACO_B200_LIB=$L DT=$DT N=$N timeout 120 python tools/kbench.py 2>&1 | tr "\n" " " >> $OUT/k.txt; echo >> $OUT/k.txt
  done; done
done; done
if [ -n "${TESTLIB:-}" ]; then TACO_B200_LIB=paper_2604_24088_b200/libtaco_b200_$TESTLIB.so timeout 900 python -m pytest tests/test_gpu_codec.py tests/test_gpu_configs.py tests/test_gpu_collective.py tests/test_gpu_reftests.py -q > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log; fi
