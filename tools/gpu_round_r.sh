mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "parity or strip or batch or graph or race or host" > gpurun_out/t_early.txt 2>&1; echo rc=$? >> gpurun_out/t_early.txt
P="cdf97/monolithic_star cdf97/sweldens/inv cdf53/monolithic cdf97/polyphase/fwd dd137/monolithic_star/fwd"
for l in base noearly; do
  if [ $l = base ]; then L=paper_1605_00561_b200/libwavelift_b200.so; else L=paper_1605_00561_b200/libwavelift_b200_$l.so; fi
  echo "== $l"; WL_LIB=$L timeout 300 python tools/size_sweep.py 4096,8192,16384 $P 2>&1 | tail -7
  WL_LIB=$L python tools/c5_breakdown.py cdf97 monolithic_star 2>&1 | tail -4
  WL_LIB=$L timeout 400 python bench.py --no-c3 --no-cpu --no-unaligned --no-dd137 --e2e-steps 0 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('value', round(d['value'],1), 'ms', round(d['ms_per_step'],4), 'c4', round(d['c4']['ms'],4), 'c5', {w: round(d['c5'][w]['ms'],2) for w in ('cdf53','cdf97')})"
done > gpurun_out/ab_early.txt 2>&1
