"""Hot SASS instructions of an ncu source page (`ncu -i X --page source --csv
--print-source sass`): top instructions by stall samples, with the dominant
stall reasons, plus totals per stall reason and per opcode class.
usage: python tools/sass_hot.py page.csv [top]"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr, data = rows[1], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = Counter()
ops = Counter()
items = []
for r in data:
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    sass = r[ix["Source"]].strip()
    op = sass.split()[0] if sass else "?"
    if op.startswith("@"):
        op = sass.split()[1]
    ops[op.split(".")[0]] += s
    per = {h: int(r[ix[h]] or 0) for h in stalls}
    tot.update(per)
    items.append((s, r[ix["Address"]][-5:], sass[:70], per))
n = sum(tot.values())
print("total samples", n)
for h, v in tot.most_common(12):
    print(f"  {h:28s} {v:7d} {100 * v / max(n, 1):5.1f}%")
print("by opcode:")
for o, v in ops.most_common(15):
    print(f"  {o:12s} {v:7d} {100 * v / max(n, 1):5.1f}%")
print("hot instructions:")
for s, a, t, per in sorted(items, key=lambda x: -x[0])[:top]:
    best = sorted(per.items(), key=lambda kv: -kv[1])[:3]
    print(f"{s:6d} {a} {t:70s} " + " ".join(f"{k[6:]}={v}" for k, v in best if v))
