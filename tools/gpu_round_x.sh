mkdir -p gpurun_out
{
for l in base ramp1 base ramp1; do
  if [ $l = base ]; then L=paper_1605_00561_b200/libwavelift_b200.so; else L=paper_1605_00561_b200/libwavelift_b200_$l.so; fi
  echo "== $l"; WL_LIB=$L timeout 300 python tools/size_sweep.py 4096,8192,16384 cdf97/monolithic_star cdf53/monolithic cdf97/sweldens/inv 2>&1 | tail -5
  WL_LIB=$L timeout 400 python bench.py --no-c3 --no-c5 --no-cpu --no-unaligned --no-dd137 --e2e-steps 0 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('value', round(d['value'],1), 'ms', round(d['ms_per_step'],4), 'c4', round(d['c4']['ms'],4))"
done
} > gpurun_out/ab_ramp.txt 2>&1
