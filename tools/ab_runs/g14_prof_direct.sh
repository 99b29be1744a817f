# ncu --set full captures of the direct-load (unaligned-shape) forwards at 8190^2 after the store work
mkdir -p gpurun_out/r02e
for p in "cdf97 monolithic_star fwd" "cdf53 monolithic fwd" "cdf97 monolithic_star inv"; do
  set -- $p
  ncu --set full --import-source on --clock-control none -k regex:'fast_kernel' -s 2 -c 1 \
      -o gpurun_out/r02e/prof_r02e_direct8190_$1_$2_$3 python tools/prof_one.py $1 $2 $3 8190 3 > /dev/null 2>&1
done
ls -la gpurun_out/r02e
