#!/bin/bash
# Round-2 geometry A/B under steady-state timing (tools/ab_steady.py).
O=gpurun_out/r02; mkdir -p $O
F53="cdf53/sweldens/fwd cdf53/iwahashi/fwd cdf53/explosive_star/fwd cdf53/monolithic/fwd cdf53/monolithic_star/fwd cdf53/polyphase/fwd cdf53/polyphase_star/fwd"
I97="cdf97/sweldens/inv cdf97/iwahashi/inv cdf97/iwahashi_star/inv cdf97/explosive/inv cdf97/monolithic/inv cdf97/monolithic_star/inv cdf97/polyphase_star/inv cdf53/monolithic/inv cdf53/sweldens/inv"
P97="cdf97/polyphase/fwd cdf97/polyphase/inv"
for n in 8192 16384; do
  python tools/ab_steady.py $n base,f53r5,f53r4,f53r4s3 $F53
  python tools/ab_steady.py $n base,i97c4,i97r6 $I97
  python tools/ab_steady.py $n base,pr2n14,pr4n8 $P97
done
