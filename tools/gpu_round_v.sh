mkdir -p gpurun_out
P="cdf53/convolution/fwd cdf97/convolution/fwd"
for l in base cm8 cm4y64; do
  if [ $l = base ]; then L=paper_1605_00561_b200/libwavelift_b200.so; else L=paper_1605_00561_b200/libwavelift_b200_$l.so; fi
  echo "== $l"; WL_LIB=$L timeout 300 python tools/size_sweep.py 8192,16384 $P 2>&1 | tail -2
done > gpurun_out/ab_conv5.txt 2>&1
