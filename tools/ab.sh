#!/bin/bash
# A/B kernel timing of variant libraries: tools/ab.sh "<programs>" tag1 tag2 ...
# (tag "" = the default library). Prints the per-program medians per variant.
progs="$1"; shift
for t in "$@"; do
  if [ -z "$t" ] || [ "$t" = base ]; then lib=paper_1605_00561_b200/libwavelift_b200.so; else lib=paper_1605_00561_b200/libwavelift_b200_$t.so; fi
  echo "== variant $t"
  WL_VERBOSE=1 WL_LIB=$lib python tools/bench_kernels.py ${SIZE:-16384} ${REPS:-15} $progs 2>&1 | grep -v "^\[wl\]" | python -c "
import sys, json
for l in sys.stdin:
    try: d=json.loads(l); print(f\"{d['program']:28s} {d['median_ms']:.4f} ms  {d['frac']:.3f}\")
    except Exception: print(l.rstrip())"
done
