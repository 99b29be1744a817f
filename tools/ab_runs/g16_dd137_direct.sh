# dd137 direct-load forwards with / without realigned stores (8190^2); dd137 unaligned parity
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity_large.py -q -k "unaligned" > gpurun_out/g16_tests.log 2>&1; echo rc=$? >> gpurun_out/g16_tests.log
sed -n '/cat > \/tmp\/ud.py/,/^PY$/p' tools/ab_runs/g10_direct97.sh | sed '1d;$d' | sed 's/for w in ("cdf97", "cdf53"):/for w in ("dd137",):/; s/wl.SCHEMES\[:9\]/wl.SCHEMES[:7]/' > /tmp/ud137.py
for i in 1 2; do python /tmp/ud137.py; WL_LIB=paper_1605_00561_b200/libwavelift_b200_nora97.so python /tmp/ud137.py; done > gpurun_out/g16_ab.txt 2>&1
