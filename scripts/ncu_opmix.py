"""SASS opcode mix of an `ncu --page source --csv` export: executed warp
instructions per opcode, normalised per `unit` threads' worth of work.

    python scripts/ncu_opmix.py prof_source.csv N_UNITS [top]
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
units = float(sys.argv[2]) / 32
top = int(sys.argv[3]) if len(sys.argv) > 3 else 20
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hi]
col = {h: i for i, h in enumerate(hdr)}
body = [r for r in rows[hi + 1:] if len(r) == len(hdr)]
c = collections.Counter()
tot = 0.0
for r in body:
    src = r[col["Source"]].split()
    if not src:
        continue
    op = (src[1] if src[0].startswith("@") else src[0]).split(".")[0]
    n = float(r[col["Instructions Executed"]] or 0)
    c[op] += n
    tot += n
for op, n in c.most_common(top):
    print(f"{op:10s} {n / units:7.1f} per warp-unit  {n / tot:5.1%}")
print(f"total {tot / units:.1f} warp instructions per 32 units")
