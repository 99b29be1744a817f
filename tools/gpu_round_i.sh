mkdir -p gpurun_out
P="cdf97/sweldens/inv cdf97/iwahashi/inv cdf97/iwahashi_star/inv cdf97/monolithic/inv cdf97/monolithic_star/inv cdf97/polyphase_star/inv"
for l in i48 i410 i58 i36; do
  L=paper_1605_00561_b200/libwavelift_b200_$l.so
  echo "== $l"; WL_VERBOSE=1 WL_LIB=$L timeout 300 python tools/size_sweep.py 8192,16384 $P 2>&1 | grep -v "^\[wl\]" | tail -8
done > gpurun_out/ab_inv97.txt 2>&1
