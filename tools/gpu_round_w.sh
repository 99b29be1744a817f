mkdir -p gpurun_out
{
for l in base ps410 ps312; do
  if [ $l = base ]; then L=paper_1605_00561_b200/libwavelift_b200.so; else L=paper_1605_00561_b200/libwavelift_b200_$l.so; fi
  echo "== $l"; WL_LIB=$L timeout 300 python tools/size_sweep.py 8192,16384 cdf97/polyphase_star/fwd 2>&1 | tail -1
done
P="dd137/sweldens/fwd dd137/iwahashi/fwd dd137/monolithic/fwd dd137/monolithic_star/fwd dd137/sweldens/inv dd137/monolithic/inv"
for m in 0x3b 0x2b 0x1b 0x0b; do echo "== mask $m"; WL_DYN_MASK=$m timeout 300 python tools/size_sweep.py 8192,16384 $P 2>&1 | tail -6; done
} > gpurun_out/ab_misc.txt 2>&1
