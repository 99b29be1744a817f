mkdir -p gpurun_out
for i in 1 2; do for t in base norev; do
  if [ $t = base ]; then L=paper_1605_00561_b200/libwavelift_b200.so; else L=paper_1605_00561_b200/libwavelift_b200_$t.so; fi
  echo "== $t"; WL_LIB=$L timeout 120 python tools/bench_step.py 20
done; done > gpurun_out/g1_step.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/g1_gputest.log 2>&1; echo rc=$? >> gpurun_out/g1_gputest.log
