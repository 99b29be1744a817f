#!/bin/bash
# Round evidence (run on the GPU box): launch list of the bench command,
# DRAM traffic per program at 8192^2, full ncu captures of the headline
# kernels. Then locally: python tools/summarize_profiles.py <tag>.
#   tools/profile_round.sh r01
set -u
TAG=${1:-r01}
O=gpurun_out
mkdir -p $O
PROGS="cdf53/sweldens cdf53/iwahashi cdf53/iwahashi_star cdf53/explosive cdf53/explosive_star cdf53/monolithic cdf53/monolithic_star cdf53/polyphase cdf53/polyphase_star cdf53/convolution cdf97/sweldens cdf97/iwahashi cdf97/iwahashi_star cdf97/explosive cdf97/explosive_star cdf97/monolithic cdf97/monolithic_star cdf97/polyphase cdf97/polyphase_star cdf97/convolution"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_$TAG.csv \
    python bench.py --steps 1 --warmup 1 --no-c3 --no-c4 --no-c5 --e2e-steps 0 --no-cpu > $O/launches_bench.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    --csv --log-file $O/traffic_$TAG.csv python tools/bench_kernels.py 8192 1 $PROGS > /dev/null 2>&1
cap() {  # name wavelet scheme dir size
    ncu --set full --import-source on --clock-control none -k regex:'fast_kernel|conv_fast' -s 2 -c 1 \
        -o $O/prof_${TAG}_$1 python tools/prof_one.py $2 $3 $4 $5 3 > /dev/null 2>&1
}
cap headline_c3_cdf97_mono_star_fwd cdf97 monolithic_star fwd 16384
cap c3_cdf97_mono_star_inv cdf97 monolithic_star inv 16384
cap c3_cdf53_mono_fwd cdf53 monolithic fwd 16384
cap c3_cdf53_mono_inv cdf53 monolithic inv 16384
cap bench_cdf97_polyphase_inv cdf97 polyphase inv 8192
ls -la $O
