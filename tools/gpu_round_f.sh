mkdir -p gpurun_out
O=paper_1605_00561_b200/libwavelift_b200_old.so
B=paper_1605_00561_b200/libwavelift_b200.so
L=paper_1605_00561_b200/libwavelift_b200_late.so
for rep in 1 2; do
  for lib in $O $B $L; do
    echo "== $lib"
    WL_LIB=$lib timeout 300 python bench.py --no-c3 --no-c5 --no-cpu --no-unaligned --no-dd137 --e2e-steps 0 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('value', round(d['value'],1), 'ms', round(d['ms_per_step'],4), 'c4', round(d['c4']['ms'],4))
ps=d['per_scheme']; print(' '.join(f'{k}:{v[0]}' for k,v in ps.items() if k.startswith('cdf97')))"
  done
done > gpurun_out/ab_bench.txt 2>&1
WL_LIB=paper_1605_00561_b200/libwavelift_b200_diaglate.so python tools/diag_times.py 8192 cdf97/monolithic_star/fwd cdf97/monolithic_star/inv cdf97/sweldens/inv cdf53/monolithic/fwd > gpurun_out/diag_late.txt 2>&1
