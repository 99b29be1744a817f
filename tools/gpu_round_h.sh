mkdir -p gpurun_out
P="cdf97/sweldens/inv cdf97/iwahashi/inv cdf97/monolithic/inv cdf97/monolithic_star/inv"
for l in old nbp_static nbp base i48 i48_static; do
  case $l in nbp_static) L=paper_1605_00561_b200/libwavelift_b200_nbp.so; E="WL_DYN=0";; i48_static) L=paper_1605_00561_b200/libwavelift_b200_i48.so; E="WL_DYN=0";; base) L=paper_1605_00561_b200/libwavelift_b200.so; E="";; *) L=paper_1605_00561_b200/libwavelift_b200_$l.so; E="";; esac
  echo "== $l"; env $E WL_LIB=$L timeout 300 python tools/size_sweep.py 8192,16384 $P 2>&1 | tail -8
done > gpurun_out/ab_bisect2.txt 2>&1
