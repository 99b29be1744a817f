mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_large.py -m gpu -q -x -k "dd137" > gpurun_out/t_dd.txt 2>&1; echo rc=$? >> gpurun_out/t_dd.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gputest5.log 2>&1; echo rc=$? >> gpurun_out/gputest5.log
python tools/size_sweep.py 4096,8192,16384 dd137/sweldens dd137/monolithic dd137/monolithic_star dd137/iwahashi dd137/explosive_star cdf97/monolithic_star cdf53/monolithic > gpurun_out/sweep_dd.txt 2>&1
ENGINE=1 python tools/size_sweep.py 2048,4096 dd137/monolithic_star >> gpurun_out/sweep_dd.txt 2>&1
