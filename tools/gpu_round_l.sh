mkdir -p gpurun_out
PART=a timeout 1500 bash tools/profile_r02.sh r02b > gpurun_out/profile_r02b_a.log 2>&1
python tools/c5_breakdown.py cdf97 monolithic_star > gpurun_out/c5_breakdown.txt 2>&1
python tools/c5_breakdown.py cdf53 monolithic_star >> gpurun_out/c5_breakdown.txt 2>&1
for l in base pc2a pc2b pc2c; do
  if [ $l = base ]; then L=paper_1605_00561_b200/libwavelift_b200.so; else L=paper_1605_00561_b200/libwavelift_b200_$l.so; fi
  echo "== $l"; WL_LIB=$L timeout 300 python tools/size_sweep.py 8192,16384 cdf97/polyphase 2>&1 | tail -2
done > gpurun_out/ab_polycpt.txt 2>&1
