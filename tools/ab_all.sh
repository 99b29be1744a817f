#!/bin/bash
# A/B of variant libraries over program sets: tools/ab_all.sh "SIZES" "PROGRAMS" tag1 tag2 ...
# (tag "cur" = the default library); prints "size lib program/dir ms" lines (tools/ab_min.py).
sizes="$1"; progs="$2"; shift 2
for S in $sizes; do
  for t in "$@"; do
    if [ "$t" = cur ]; then L=paper_1605_00561_b200/libwavelift_b200.so; else L=paper_1605_00561_b200/libwavelift_b200_$t.so; fi
    WL_LIB=$L timeout 200 python tools/ab_min.py $S ${REPS:-11} $progs | sed "s/^/$S /"
  done
done
