# CPT = 4 direct-load inverse (cdf97 Polyphase) vector row stores: parity + A/B, full GPU tests
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/g13_gputest.log 2>&1; echo rc=$? >> gpurun_out/g13_gputest.log
sed -n '/cat > \/tmp\/uinv.py/,/^PY$/p' tools/ab_runs/g8_invpair.sh | sed '1d;$d' > /tmp/uinv.py
for i in 1 2; do python /tmp/uinv.py; WL_LIB=paper_1605_00561_b200/libwavelift_b200_noinvp.so python /tmp/uinv.py; done > gpurun_out/g13_ab.txt 2>&1
