mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputest3.log 2>&1; echo rc=$? >> gpurun_out/gputest3.log
P="cdf53/monolithic cdf97/monolithic_star cdf97/sweldens cdf97/iwahashi/inv cdf97/polyphase/fwd cdf97/convolution/fwd cdf53/convolution/fwd"
python tools/size_sweep.py 4096,8192,16384 $P > gpurun_out/sweep_dyn.txt 2>&1
WL_DYN=0 python tools/size_sweep.py 4096,8192,16384 $P > gpurun_out/sweep_static.txt 2>&1
WL_LIB=paper_1605_00561_b200/libwavelift_b200_diag.so python tools/diag_times.py 8192 cdf97/monolithic_star/fwd cdf97/monolithic_star/inv cdf97/sweldens/inv cdf53/monolithic/fwd > gpurun_out/diag_dyn.txt 2>&1
