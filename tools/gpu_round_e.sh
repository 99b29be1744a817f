mkdir -p gpurun_out
P="dd137/sweldens dd137/monolithic dd137/monolithic_star dd137/iwahashi dd137/explosive_star"
for l in base g66 i284 i266 g58; do
  if [ $l = base ]; then L=paper_1605_00561_b200/libwavelift_b200.so; else L=paper_1605_00561_b200/libwavelift_b200_$l.so; fi
  echo "== $l"; WL_LIB=$L timeout 300 python tools/size_sweep.py 8192,16384 $P 2>&1 | tail -12
done > gpurun_out/ab_dd.txt 2>&1
