# after adopting 3-row direct-load warps + realigned stores for cdf97: tests, timing, bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/g11_gputest.log 2>&1; echo rc=$? >> gpurun_out/g11_gputest.log
sed -n '/cat > \/tmp\/ud.py/,/^PY$/p' tools/ab_runs/g10_direct97.sh | sed '1d;$d' > /tmp/ud.py
python /tmp/ud.py > gpurun_out/g11_direct.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g11_smoke.log 2>&1
timeout 400 python bench.py > gpurun_out/g11_bench.json 2> gpurun_out/g11_bench.err
