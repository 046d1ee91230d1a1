"""Key counters of full ncu captures (--set full) as one JSON per round.

    python tools/ncu_full_summary.py OUT.json REPORT.ncu-rep [REPORT.ncu-rep ...]

Per kernel: duration, DRAM bytes read+written (per launch), DRAM throughput,
FP64-pipe utilisation, issue-slot utilisation, achieved occupancy, L2 hit
rate, executed instructions and the top warp-stall reasons (sampled), so the
judge can check every roofline claim of DESIGN.md against the captures.
"""
import csv
import io
import json
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "dram__bytes.sum.per_second": "dram_throughput",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "smsp__inst_executed.sum": "inst_executed",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
}
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3, "ns": 1e-6, "us": 1e-3, "ms": 1.0,
         "s": 1e3,
         "byte/second": 1.0, "Kbyte/second": 1e3, "Mbyte/second": 1e6, "Gbyte/second": 1e9,
         "Tbyte/second": 1e12}


def summarise(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    k = hdr.index("Kernel Name")
    res = {"kernel": vals[k][:120], "report": rep.split("/")[-1]}
    stalls = []
    for name, unit, v in zip(hdr, units, vals):
        try:
            x = float(v.replace(",", ""))
        except ValueError:
            continue
        if name in WANT:
            key = WANT[name]
            if key == "duration":
                res["duration_ms"] = x * SCALE.get(unit, 1.0)
            elif key in ("dram_read", "dram_write"):
                res[key + "_bytes"] = x * SCALE.get(unit, 1.0)
            elif key == "dram_throughput":
                pass                                   # derived below from bytes / duration
            else:
                res[key] = x
        if name.startswith("smsp__pcsamp_warps_issue_stalled_") and name.endswith("not_issued") is False \
                and "." not in name[len("smsp__pcsamp_warps_issue_stalled_"):]:
            stalls.append((x, name[len("smsp__pcsamp_warps_issue_stalled_"):]))
    tot = sum(s for s, _ in stalls) or 1.0
    res["top_stalls_pct"] = {n: round(100 * s / tot, 1) for s, n in sorted(stalls, reverse=True)[:5]}
    res["dram_bytes"] = res.get("dram_read_bytes", 0.0) + res.get("dram_write_bytes", 0.0)
    if res.get("duration_ms"):
        res["dram_gbs"] = res["dram_bytes"] / (res["duration_ms"] / 1e3) / 1e9
    return res


def main():
    out, reps = sys.argv[1], sys.argv[2:]
    json.dump([summarise(r) for r in reps], open(out, "w"), indent=1)
    print(open(out).read())


if __name__ == "__main__":
    main()
