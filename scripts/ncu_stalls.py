"""Stall breakdown of an `ncu -i REP --page source --csv` export (SASS view):
total samples per stall reason and the top-N instructions by samples.

    python scripts/ncu_stalls.py prof_source.csv [N]
"""
import csv
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 15
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hdr_i]
    body = [r for r in rows[hdr_i + 1:] if len(r) == len(hdr)]
    col = {h: i for i, h in enumerate(hdr)}
    stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]

    def num(r, h):
        try:
            return float(r[col[h]] or 0)
        except ValueError:
            return 0.0
    tot = {h: sum(num(r, h) for r in body) for h in stall_cols}
    all_s = sum(tot.values()) or 1
    print("samples", int(all_s), "instructions executed",
          int(sum(num(r, "Instructions Executed") for r in body)))
    for h, v in sorted(tot.items(), key=lambda kv: -kv[1])[:10]:
        print(f"  {h:28s} {v / all_s:6.1%}")
    key = "Warp Stall Sampling (All Samples)"
    print(f"top {top} instructions:")
    for r in sorted(body, key=lambda r: -num(r, key))[:top]:
        reasons = sorted(((num(r, h), h) for h in stall_cols), reverse=True)[:2]
        print(f"  {num(r, key) / all_s:6.1%} {r[col['Address']]:>6s} {r[col['Source']][:60]:60s} "
              + " ".join(f"{h[6:]}={v / all_s:.1%}" for v, h in reasons))


if __name__ == "__main__":
    main()
