mkdir -p gpurun_out
run() {  # tag lib mask
  echo "== $1 mask $3"; WL_LIB=$2 WL_DYN_MASK=$3 timeout 400 python bench.py --no-c5 --no-cpu --no-unaligned --no-dd137 --e2e-steps 0 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('value', round(d['value'],1), 'ms', round(d['ms_per_step'],4), 'c4', round(d['c4']['ms'],4))
print('c3', {k: v[0] for k, v in d['north_star']['c3'].items()})
ps=d['per_scheme']; print(' '.join(f'{k}:{v[0]}' for k,v in ps.items() if k.endswith('fwd')))"
}
B=paper_1605_00561_b200/libwavelift_b200.so
for m in 0x0 0x1 0x3 0x3f; do run base $B $m; done
for v in f410 f312 f53r4; do run $v paper_1605_00561_b200/libwavelift_b200_$v.so 0x0; done
run base $B 0x0
