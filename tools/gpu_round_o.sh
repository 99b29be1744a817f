mkdir -p gpurun_out
P="dd137/sweldens/fwd dd137/iwahashi/fwd dd137/monolithic/fwd dd137/monolithic_star/fwd dd137/explosive_star/fwd"
for l in base f137a f137b f137c; do
  if [ $l = base ]; then L=paper_1605_00561_b200/libwavelift_b200.so; else L=paper_1605_00561_b200/libwavelift_b200_$l.so; fi
  echo "== $l"; WL_VERBOSE=1 WL_LIB=$L timeout 300 python tools/size_sweep.py 8192,16384 $P 2>&1 | grep -v "^\[wl\]" | tail -5
done > gpurun_out/ab_dd_fwd.txt 2>&1
