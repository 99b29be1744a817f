mkdir -p gpurun_out
for l in base m58 m48; do
  if [ $l = base ]; then L=paper_1605_00561_b200/libwavelift_b200.so; else L=paper_1605_00561_b200/libwavelift_b200_$l.so; fi
  echo "== $l"; WL_LIB=$L timeout 300 python tools/size_sweep.py 8192,16384 cdf97/monolithic/inv cdf97/monolithic_star/inv cdf97/sweldens/inv 2>&1 | tail -3
done > gpurun_out/ab_mono.txt 2>&1
for m in 0x3f 0x3b 0x2a 0x00 0x0b; do
  echo "== mask $m"; WL_DYN_MASK=$m timeout 300 python bench.py --no-c3 --no-c5 --no-cpu --no-unaligned --no-dd137 --e2e-steps 0 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('value', round(d['value'],1), 'ms', round(d['ms_per_step'],4), 'c4', round(d['c4']['ms'],4))"
done > gpurun_out/ab_mask.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "parity or strip or batch or graph or race" > gpurun_out/t_geo.txt 2>&1; echo rc=$? >> gpurun_out/t_geo.txt
