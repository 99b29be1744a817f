# cdf97 Polyphase: two CTAs of 5 compute warps (3-row warps) per SM vs one CTA of 10
mkdir -p gpurun_out
for S in 8192 16384; do SIZE=$S bash tools/ab.sh "cdf97/polyphase" base p3x5 base p3x5; done > gpurun_out/g3_kern.txt 2>&1
