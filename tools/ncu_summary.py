"""Summarise an ncu launch list (gpu__time_duration + dram bytes per launch).

    python tools/ncu_summary.py LAUNCHES.csv OUT_SUMMARY.txt [OUT_TRAFFIC.json] [header line] [config key]

Writes per-kernel launch counts, summed time, step share and DRAM bytes per
launch; the optional JSON maps the bench's profiler names of the dominant
kernels to DRAM bytes per launch (bench.py's roofline.traffic).
"""
import collections
import csv
import json
import re
import sys

# bench profiler name -> ncu kernel name prefix
PROFILER_NAMES = {"trsv_ilu": ("k_wf_pf", "k_wf", "k_tile_flow"), "gs_dots2": ("k_dots2",), "gs_axpy2": ("k_axpy2",),
                  "spmv_A": ("k_spmv_sell",), "trsv_ic_pair": ("k_chain_pair",)}


def main():
    src, out = sys.argv[1], sys.argv[2]
    traffic_out = sys.argv[3] if len(sys.argv) > 3 else None
    header = sys.argv[4] if len(sys.argv) > 4 else ""
    cfg_key = sys.argv[5] if len(sys.argv) > 5 else "config5"
    rows = list(csv.reader(open(src)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mn, mv, idi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per, names = collections.defaultdict(dict), {}
    for r in rows[hi + 1:]:
        if len(r) <= mv:
            continue
        per[r[idi]][r[mn]] = float(r[mv].replace(",", ""))
        names[r[idi]] = r[ki]
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    tot = 0.0
    for i, m in per.items():
        nm = re.search(r"(k_\w+|DeviceScan\w*|DeviceRadix\w*|DeviceSelect\w*|\w+Kernel\w*)", names[i])
        key = nm.group(1) if nm else names[i][:40]
        t = m.get("gpu__time_duration.sum", 0.0)
        b = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        a = agg[key]
        a[0] += 1
        a[1] += t
        a[2] += b
        tot += t
    with open(out, "w") as f:
        f.write(header + "\n" if header else "")
        f.write("# ncu launch list (cold cache, serialised launches: compare SHARES, not absolute times)\n")
        f.write(f"# launches {len(per)}  total {tot / 1e6:.3f} ms\n")
        f.write(f"{'kernel':34s} {'launches':>8s} {'ms':>10s} {'share%':>7s} {'DRAM MB/launch':>15s} {'GB/s':>8s}\n")
        for k, (n, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            f.write(f"{k:34s} {n:8d} {t / 1e6:10.3f} {t / tot * 100:7.2f} {b / n / 1e6:15.2f} "
                    f"{(b / t if t else 0):8.1f}\n")
    if traffic_out:
        tr = {}
        for prof, kerns in PROFILER_NAMES.items():
            hit = [(n, b) for k, (n, t, b) in agg.items() if k in kerns]
            if hit:
                n = sum(x[0] for x in hit)
                tr[prof] = sum(x[1] for x in hit) / n
        try:
            allcfg = json.load(open(traffic_out))
            if not all(isinstance(v, dict) for v in allcfg.values()):
                allcfg = {}
        except Exception:
            allcfg = {}
        allcfg[cfg_key] = tr
        json.dump(allcfg, open(traffic_out, "w"), indent=1)
    print(open(out).read())


if __name__ == "__main__":
    main()
