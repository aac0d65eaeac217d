mkdir -p gpurun_out/r2m
for v in default f3 f3np f0np; do
  if [ $v = default ]; then L=paper_2604_24088_b200/libtaco_b200.so; else L=paper_2604_24088_b200/libtaco_b200_$v.so; fi
  echo "== $v" >> gpurun_out/r2m/peer.txt
  TACO_B200_LIB=$L REPS=100 timeout 300 python tools/peer_prof.py >> gpurun_out/r2m/peer.txt 2>&1
  TACO_B200_LIB=$L ITERS=2 REPS=2 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k[123]x" --csv --log-file gpurun_out/r2m/launch_$v.csv python tools/peer_prof.py > /dev/null 2>&1
done
