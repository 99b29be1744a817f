#!/bin/bash
# Round evidence (tag = $1, default r02) (run on the GPU box): launch list of the bench step, DRAM
# traffic per program at 8192^2 and for the configs[2] programs at 16384^2,
# full ncu captures of the kernels the bench line and VERDICT name.
# Then locally: python tools/summarize_r02.py
set -u
TAG=${1:-r02}
O=gpurun_out/$TAG
mkdir -p $O
PROGS="cdf53/sweldens cdf53/iwahashi cdf53/iwahashi_star cdf53/explosive cdf53/explosive_star cdf53/monolithic cdf53/monolithic_star cdf53/polyphase cdf53/polyphase_star cdf53/convolution cdf97/sweldens cdf97/iwahashi cdf97/iwahashi_star cdf97/explosive cdf97/explosive_star cdf97/monolithic cdf97/monolithic_star cdf97/polyphase cdf97/polyphase_star cdf97/convolution"
C3="cdf97/monolithic_star cdf97/monolithic cdf97/sweldens cdf53/monolithic cdf53/monolithic_star"
# PART=a: launch list, traffic, first captures; PART=b: the other captures
# (each part's output stays under gpurun's 64 MiB copy-back limit)
PART=${PART:-a}
if [ "$PART" = a ]; then
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_$TAG.csv \
    python bench.py --steps 1 --warmup 3 --no-c3 --no-c4 --no-c5 --e2e-steps 0 --no-cpu --no-unaligned --no-dd137 > $O/launches_bench.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    --csv --log-file $O/traffic_$TAG.csv python tools/bench_kernels.py 8192 1 $PROGS > /dev/null 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    --csv --log-file $O/traffic_c3_$TAG.csv python tools/bench_kernels.py 16384 1 $C3 > /dev/null 2>&1
fi
cap() {  # name wavelet scheme dir size
    ncu --set full --import-source on --clock-control none -k regex:'fast_kernel|conv_fast' -s 2 -c 1 \
        -o $O/prof_${TAG}_$1 python tools/prof_one.py $2 $3 $4 $5 3 > /dev/null 2>&1
}
if [ "$PART" = a ]; then
cap bench_cdf97_sweldens_inv cdf97 sweldens inv 8192
cap bench_cdf97_polyphase_fwd cdf97 polyphase fwd 8192
cap bench_cdf97_convolution_fwd cdf97 convolution fwd 8192
else
cap bench_cdf97_iwahashi_fwd cdf97 iwahashi fwd 8192
cap bench_dd137_monolithic_star_fwd dd137 monolithic_star fwd 8192
cap c3_cdf97_mono_star_fwd cdf97 monolithic_star fwd 16384
cap c3_cdf97_sweldens_inv cdf97 sweldens inv 16384
fi
ls -la $O | tail -20
