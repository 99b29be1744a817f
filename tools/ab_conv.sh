#!/bin/bash
# conv row-segment loads: shuffles (base) vs overlapping 8-byte loads (conv0)
for n in 8192 16384; do
  python tools/ab_steady.py $n base,conv0 cdf53/convolution/fwd cdf97/convolution/fwd
done
