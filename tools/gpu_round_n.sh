mkdir -p gpurun_out
for l in base npf base npf; do
  if [ $l = base ]; then L=paper_1605_00561_b200/libwavelift_b200.so; else L=paper_1605_00561_b200/libwavelift_b200_$l.so; fi
  echo "== $l"
  WL_LIB=$L timeout 400 python bench.py --no-c3 --no-cpu --no-unaligned --no-dd137 --e2e-steps 0 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('value', round(d['value'],1), 'ms', round(d['ms_per_step'],4), 'c4', round(d['c4']['ms'],4), 'c5', {w: round(d['c5'][w]['ms'],2) for w in ('cdf53','cdf97')})"
  WL_LIB=$L python tools/c5_breakdown.py cdf97 monolithic_star 2>&1 | tail -4
done > gpurun_out/ab_prefetch.txt 2>&1
timeout 600 python -m pytest tests -m gpu -q -x -k "race or parity_large or strip" > gpurun_out/t_pf.txt 2>&1; echo rc=$? >> gpurun_out/t_pf.txt
