mkdir -p gpurun_out
P="cdf97/sweldens/fwd cdf97/iwahashi/fwd cdf97/monolithic/fwd cdf97/monolithic_star/fwd cdf97/explosive_star/fwd cdf97/polyphase_star/fwd cdf53/monolithic/fwd"
for l in base c97f2a c97f2b; do
  if [ $l = base ]; then L=paper_1605_00561_b200/libwavelift_b200.so; else L=paper_1605_00561_b200/libwavelift_b200_$l.so; fi
  echo "== $l"; WL_VERBOSE=1 WL_LIB=$L timeout 300 python tools/size_sweep.py 8192,16384 $P 2>&1 | grep -v "^\[wl\]" | tail -7
done > gpurun_out/ab_c97f2.txt 2>&1
