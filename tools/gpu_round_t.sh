mkdir -p gpurun_out
P="cdf53/sweldens/fwd cdf53/iwahashi/fwd cdf53/monolithic/fwd cdf53/monolithic_star/fwd cdf53/polyphase/fwd cdf53/polyphase_star/fwd cdf53/explosive_star/fwd"
for l in base f53r4 f53r3n2; do
  if [ $l = base ]; then L=paper_1605_00561_b200/libwavelift_b200.so; else L=paper_1605_00561_b200/libwavelift_b200_$l.so; fi
  echo "== $l"; WL_LIB=$L timeout 300 python tools/size_sweep.py 8192,16384 $P 2>&1 | tail -7
  WL_LIB=$L python tools/c5_breakdown.py cdf53 monolithic_star 2>&1 | tail -1
done > gpurun_out/ab_f53.txt 2>&1
