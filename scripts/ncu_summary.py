"""Summarise an ncu report (--set full) of the step kernel into JSON.

    python scripts/ncu_summary.py gpurun_out/r1b/prof_step.ncu-rep [n_fn] > out.json
    python scripts/ncu_summary.py gpurun_out/r1c/prof_step_f32_raw.csv [n_fn] > out.json

Reads `ncu -i --page raw --csv`; reports duration, DRAM bytes (read/write)
per launch, throughput, L1/L2 sector counts and hit rates, occupancy and
registers -- and, given n_fn, DRAM bytes per fluid node vs the 304 B (fp64) / 152 B (fp32) model.
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_peak",
    "lts__t_sectors_srcunit_tex_op_read.sum": "l2_read_sectors_from_sm",
    "lts__t_sectors_srcunit_tex_op_write.sum": "l2_write_sectors_from_sm",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum": "l1_ld_sectors",
    "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum": "l1_ld_requests",
    "l1tex__t_sector_hit_rate.pct": "l1_hit_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "launch__registers_per_thread": "registers",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "sm__maximum_warps_per_active_cycle_pct": "theoretical_occupancy_pct",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "smsp__inst_executed.sum": "instructions",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio": "stall_long_sb",
}
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12,
         "ms": 1e-3, "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9,
         "nsecond": 1e-9, "s": 1.0}


def main():
    rep = sys.argv[1]
    n_fn = int(sys.argv[2]) if len(sys.argv) > 2 else None
    if rep.endswith(".csv"):           # a `--page raw --csv` export made on the GPU box
        raw = open(rep).read()
    else:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        rec = {"kernel": vals[hdr.index("Kernel Name")][:120]}
        for k, name in KEYS.items():
            if k in hdr:
                i = hdr.index(k)
                v = vals[i].replace(",", "")
                try:
                    v = float(v) * SCALE.get(units[i], 1.0)
                except ValueError:
                    pass
                rec[name] = v
        if "dram_read" in rec and "dram_write" in rec:
            rec["dram_bytes"] = rec["dram_read"] + rec["dram_write"]
            if "duration" in rec:
                rec["dram_gbs"] = rec["dram_bytes"] / rec["duration"] / 1e9
            if n_fn:
                rec["dram_bytes_per_node"] = rec["dram_bytes"] / n_fn
                rec["algorithmic_bytes_per_node"] = 152 if "<float" in rec.get("kernel", "") else 304
        out.append(rec)
    json.dump(out, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
