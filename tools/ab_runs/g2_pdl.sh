# PDL re-measurement (round 1: 3.7% slower before dynamic claims)
mkdir -p gpurun_out
for i in 1 2; do for t in base pdl; do
  if [ $t = base ]; then L=paper_1605_00561_b200/libwavelift_b200.so; else L=paper_1605_00561_b200/libwavelift_b200_$t.so; fi
  echo "== $t"; WL_LIB=$L timeout 120 python tools/bench_step.py 20
done; done > gpurun_out/g2_step.txt 2>&1
SIZE=8192 bash tools/ab.sh "cdf97/sweldens cdf97/monolithic cdf53/monolithic cdf97/polyphase" base pdl > gpurun_out/g2_kern.txt 2>&1
