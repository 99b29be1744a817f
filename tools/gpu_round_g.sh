mkdir -p gpurun_out
P="cdf97/sweldens cdf97/iwahashi/inv cdf97/monolithic/inv cdf97/monolithic_star/inv cdf97/monolithic/fwd"
for l in old base nb np nbp base_static; do
  case $l in base) L=paper_1605_00561_b200/libwavelift_b200.so; E="";; base_static) L=paper_1605_00561_b200/libwavelift_b200.so; E="WL_DYN=0";; *) L=paper_1605_00561_b200/libwavelift_b200_$l.so; E="";; esac
  echo "== $l"; env $E WL_LIB=$L timeout 300 python tools/size_sweep.py 8192,16384 $P 2>&1 | tail -8
done > gpurun_out/ab_bisect.txt 2>&1
