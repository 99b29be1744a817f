"""Summarise tools/ab_all.sh output: per size and program/dir, each variant's
median ms relative to 'libwavelift_b200.so'; totals per direction.
usage: python tools/ab_table.py FILE [fwd|inv]"""
import collections
import sys

d = collections.defaultdict(dict)
for line in open(sys.argv[1]):
    p = line.split()
    if len(p) == 5 and p[4] == "ms":
        d[(p[0], p[2])][p[1].replace("libwavelift_b200", "").replace(".so", "") or "cur"] = float(p[3])
want = sys.argv[2] if len(sys.argv) > 2 else None
libs = sorted({k for v in d.values() for k in v}, key=lambda x: (x != "cur", x))
print("size  program".ljust(34) + "".join(x.rjust(9) for x in libs))
tot = collections.defaultdict(float)
for (S, pr), v in sorted(d.items(), key=lambda x: (int(x[0][0]), x[0][1])):
    if want and not pr.endswith(want):
        continue
    print(f"{S:5s} {pr:28s}" + "".join(f"{v.get(l, float('nan')):9.4f}" for l in libs))
    for l in libs:
        tot[(S, l)] += v.get(l, 0.0)
for S in sorted({k[0] for k in tot}, key=int):
    print(f"{S:5s} {'total':28s}" + "".join(f"{tot[(S, l)]:9.4f}" for l in libs))
