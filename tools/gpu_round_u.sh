mkdir -p gpurun_out
P="cdf53/sweldens/inv cdf53/iwahashi/inv cdf53/monolithic/inv cdf53/monolithic_star/inv cdf53/polyphase/inv cdf53/explosive/inv cdf53/polyphase_star/inv"
for l in base i53r4 i53r5; do
  if [ $l = base ]; then L=paper_1605_00561_b200/libwavelift_b200.so; else L=paper_1605_00561_b200/libwavelift_b200_$l.so; fi
  echo "== $l"; WL_VERBOSE=1 WL_LIB=$L timeout 300 python tools/size_sweep.py 8192,16384 $P 2>&1 | grep -v "^\[wl\]" | tail -7
done > gpurun_out/ab_i53.txt 2>&1
