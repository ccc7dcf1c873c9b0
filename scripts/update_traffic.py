"""Record the step kernel's DRAM traffic per launch for bench.py's
roofline.traffic, keyed to the current kernel sources.

    python scripts/update_traffic.py KEY RAW_CSV [capture-note]

RAW_CSV is an `ncu -i <rep> --page raw --csv` export of one `--set full`
capture of the bench's step kernel (scripts/traffic_capture.sh makes it on
the GPU box).  KEY is the bench line's `<workload>_<table>` (e.g.
channel256_periodic_f64_b200).  bench.py uses the entry only while
bench.kernel_source_hash() still equals the recorded src_sha, so a kernel
change turns the figure into null ("stale") instead of a wrong number.
"""
import csv
import io
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12}


def dram_bytes(raw):
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        if "step_kernel" not in vals[hdr.index("Kernel Name")]:
            continue
        tot = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = hdr.index(k)
            tot += float(vals[i].replace(",", "")) * SCALE.get(units[i], 1.0)
        out.append(tot)
    if not out:
        raise SystemExit("no step_kernel row in the export")
    return sum(out) / len(out)


def main():
    key, path = sys.argv[1], sys.argv[2]
    note = sys.argv[3] if len(sys.argv) > 3 else os.path.basename(path)
    dst = os.path.join(ROOT, "profiles", "roofline_traffic.json")
    d = json.load(open(dst)) if os.path.exists(dst) else {}
    d = {k: v for k, v in d.items() if isinstance(v, dict) or k == "_note"}
    d["_note"] = ("dram__bytes_read.sum + dram__bytes_write.sum per launch of step_kernel from "
                  "one ncu --set full capture; bench.py uses an entry only while src_sha equals "
                  "the hash of the current kernel sources (bench.KERNEL_SOURCES)")
    d[key] = {"traffic": dram_bytes(open(path).read()), "src_sha": bench.kernel_source_hash(),
              "capture": note}
    json.dump(d, open(dst, "w"), indent=1)
    print(json.dumps(d[key]))


if __name__ == "__main__":
    main()
