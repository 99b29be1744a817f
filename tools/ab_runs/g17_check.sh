# final check: full GPU tests, smoke, bench at HEAD
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/g17_gputest.log 2>&1; echo rc=$? >> gpurun_out/g17_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g17_smoke.log 2>&1
timeout 400 python bench.py > gpurun_out/g17_bench.json 2> gpurun_out/g17_bench.err
