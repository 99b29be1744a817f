mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "unaligned or direct or strip" > gpurun_out/t_direct3.txt 2>&1; echo rc=$? >> gpurun_out/t_direct3.txt
for l in base; do
  if [ $l = base ]; then L=paper_1605_00561_b200/libwavelift_b200.so; else L=paper_1605_00561_b200/libwavelift_b200_$l.so; fi
  echo "== $l"; WL_LIB=$L timeout 400 python bench.py --no-c3 --no-c4 --no-c5 --no-cpu --no-dd137 --e2e-steps 0 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('value', round(d['value'],1)); print({k: v['ms'] for k, v in d['unaligned'].items()})"
  ENGINE=3 WL_LIB=$L timeout 300 python tools/size_sweep.py 4096,8192 cdf97/monolithic_star cdf53/monolithic cdf97/polyphase dd137/sweldens 2>&1 | tail -8
done > gpurun_out/ab_direct3.txt 2>&1
