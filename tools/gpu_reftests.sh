#!/usr/bin/env bash
# run the reference's own unit tests + acceptance gate relinked against libtaco_b200.so
OUT=gpurun_out/${1:-reftests}; mkdir -p $OUT
for t in oracle/_ref/reftest_test_*; do timeout 600 $t > $OUT/$(basename $t).log 2>&1; echo "rc=$?" >> $OUT/$(basename $t).log; done
for c in 1 2 3 4 5 6 7 8 9; do timeout 600 oracle/_ref/reftest_acceptance --criterion $c > $OUT/acceptance_$c.log 2>&1; echo "rc=$?" >> $OUT/acceptance_$c.log; done
