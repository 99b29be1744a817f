mkdir -p gpurun_out
P="cdf97/monolithic_star cdf97/sweldens/inv cdf53/monolithic/fwd cdf97/polyphase/fwd"
for l in base nowrap; do
  if [ $l = base ]; then L=paper_1605_00561_b200/libwavelift_b200.so; else L=paper_1605_00561_b200/libwavelift_b200_$l.so; fi
  echo "== $l"; WL_LIB=$L timeout 300 python tools/size_sweep.py 4096,8192,16384 $P 2>&1 | tail -5
  WL_LIB=$L python tools/c5_breakdown.py cdf97 monolithic_star 2>&1 | tail -4
done > gpurun_out/ab_nowrap.txt 2>&1
