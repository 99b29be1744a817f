mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "polyphase or sass or race" > gpurun_out/t_pm.txt 2>&1; echo rc=$? >> gpurun_out/t_pm.txt
for n in 8192 16384; do for l in base pm0 pmr4 pmr2; do python tools/ab_steady.py $n $l cdf97/polyphase cdf97/polyphase_star/fwd; done; done > gpurun_out/ab_pm.txt 2>&1
