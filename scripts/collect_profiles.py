"""Copy one evidence pass (scripts/profile_round.sh TAG, merged back into
gpurun_out/TAG/) into profiles/ as TAG_* files, with the ncu captures
summarised to JSON (scripts/ncu_summary.py) and the sparse DRAM counts
collected into TAG_ncu_sparse_dram.json.  Updates roofline_traffic.json,
which bench.py reports as roofline.traffic.

    python scripts/collect_profiles.py r1d
"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
N_CHANNEL = 256 ** 3
N_PACK02 = 3429472


def main():
    tag = sys.argv[1]
    src = os.path.join(ROOT, "gpurun_out", tag)
    dst = os.path.join(ROOT, "profiles")
    out = lambda name: os.path.join(dst, f"{tag}_{name}")  # noqa: E731
    copies = {"bench.json": "bench_n1.json", "bench_f32.json": "bench_n1_f32.json",
              "bench_fma.json": "bench_n1_fma.json", "bench_ref.json": "bench_reference.json",
              "sweep.jsonl": "porosity_sweep.jsonl", "halo_overhead.jsonl": "halo_overhead.jsonl",
              "cavity64.jsonl": "cavity64.jsonl", "launches.csv": "launches_channel256_f64.csv",
              "memcheck.txt": "memcheck.txt", "racecheck.txt": "racecheck.txt",
              "smoke.txt": "smoke.txt"}
    for a, b in copies.items():
        if os.path.exists(os.path.join(src, a)):
            shutil.copy(os.path.join(src, a), out(b))
    with open(out("ladder.jsonl"), "w") as f:
        for name in ("ladder_f64.jsonl", "ladder_f64_fma.jsonl", "ladder_f32.jsonl"):
            p = os.path.join(src, name)
            if os.path.exists(p):
                f.write(open(p).read())
    lines = open(os.path.join(src, "pytest_gpu.txt")).read().splitlines()
    open(out("pytest_gpu_summary.txt"), "w").write("\n".join(lines[-3:]) + "\n")
    summ = os.path.join(ROOT, "scripts", "ncu_summary.py")
    for k, n, name in (("f64", N_CHANNEL, "ncu_step_channel256_f64"),
                       ("f32", N_CHANNEL, "ncu_step_channel256_f32"),
                       ("mrt", N_CHANNEL, "ncu_step_channel256_mrt"),
                       ("mrt_fma", N_CHANNEL, "ncu_step_channel256_mrt_fma"),
                       ("compact_p02", N_PACK02, "ncu_step_spheres_p02_compact_f64")):
        raw = os.path.join(src, f"prof_step_{k}_raw.csv")
        if not os.path.exists(raw):
            continue
        js = subprocess.run([sys.executable, summ, raw, str(n)], capture_output=True,
                            text=True, check=True).stdout
        open(out(name + ".json"), "w").write(js)
        det = os.path.join(src, f"prof_step_{k}_details.txt")
        if os.path.exists(det):
            shutil.copy(det, out(name + "_details.txt"))
    sweep = [json.loads(l) for l in open(os.path.join(src, "sweep.jsonl")) if l.startswith("{")]
    sparse = {}
    for st in ("blocks", "compact"):
        for p in ("0.2", "0.5", "0.9"):
            fn = os.path.join(src, f"ncu_sparse_{st}_p{p}.csv")
            if not os.path.exists(fn):
                continue
            txt = open(fn).read()
            rows = list(csv.reader(io.StringIO(txt[txt.index('"ID"'):])))
            v = {}
            for r in rows[1:]:
                d = dict(zip(rows[0], r))
                v[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
            n = [r["n_fn"] for r in sweep if r["case"] == f"spheres_p{p}"
                 and r["precision"] == "f64" and r["storage"] == st][0]
            b = v["dram__bytes_read.sum"] + v["dram__bytes_write.sum"]
            sparse[f"spheres_p{p}_{st}"] = {
                "n_fn": n, "dram_read": v["dram__bytes_read.sum"],
                "dram_write": v["dram__bytes_write.sum"], "duration_ns": v["gpu__time_duration.sum"],
                "dram_bytes_per_node": b / n, "model_bytes_per_node": 304, "overfetch": b / n / 304}
    json.dump(sparse, open(out("ncu_sparse_dram.json"), "w"), indent=1)
    t_path = os.path.join(dst, "roofline_traffic.json")
    t = json.load(open(t_path))
    for key, name in (("channel256_f64_b200", "ncu_step_channel256_f64"),
                      ("channel256_f32_b200", "ncu_step_channel256_f32")):
        p = out(name + ".json")
        if os.path.exists(p):
            t[key] = json.load(open(p))[0]["dram_bytes"]
    t["_note"] = ("dram__bytes_read.sum + dram__bytes_write.sum per launch of step_kernel from "
                  f"one ncu --set full capture (profiles/{tag}_ncu_step_channel256_*.json); "
                  "bench.py reads this as roofline.traffic")
    json.dump(t, open(t_path, "w"), indent=1)
    print(f"collected {tag}")


if __name__ == "__main__":
    main()
