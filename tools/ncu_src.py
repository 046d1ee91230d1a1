"""Summarise an ncu source page (per-line warp-stall samples) for one kernel.

    python tools/ncu_src.py REPORT.ncu-rep KERNEL_REGEX [N]
"""
import csv
import io
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", 
                          "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    start = next(i for i, r in enumerate(rows) if r and r[0] in ("Line", "#", "Address"))
    hdr = rows[start]
    si = hdr.index("Source")
    wi = hdr.index("Warp Stall Sampling (All Samples)")
    stalls = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    data = []
    for r in rows[start + 1:]:
        if len(r) <= wi or not r[wi]:
            continue
        try:
            w = float(r[wi])
        except ValueError:
            continue
        if w <= 0:
            continue
        br = sorted(((float(r[i] or 0), hdr[i][6:]) for i in stalls), reverse=True)[:3]
        data.append((w, r[0], r[si].strip()[:90], br))
    tot = sum(d[0] for d in data) or 1
    for w, line, src, br in sorted(data, reverse=True)[:top]:
        s = ", ".join(f"{n}={v / w * 100:.0f}%" for v, n in br if v > 0)
        print(f"{w / tot * 100:5.1f}%  {line:>5}  {src:90s}  [{s}]")


if __name__ == "__main__":
    main()
