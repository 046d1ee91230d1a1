"""Step timeline of the axial pencil solve (EDFA_AX_DEBUG dump of the last
solve): per block, first/last step time and the mean step duration."""
import os, subprocess, sys
import numpy as np
path = "/tmp/axdbg.txt"
if len(sys.argv) < 2:
    env = dict(os.environ, EDFA_AX_DEBUG=path)
    subprocess.run([sys.executable, "tools/tiledbg.py"], env=env, check=True)
with open(path) as f:
    NJ, NK, ns = map(int, f.readline().split())
    d = np.array([int(x) for x in f], dtype=np.int64).reshape(NJ * NK, ns)
t0 = d.min()
d = (d - d[:, :1]) / 1965.0  # cycles -> us (per-SM clocks: block-relative)
print("span us %.2f" % d.max())
for blk in [0, 1, 2, NJ, NJ + 1, 2 * NJ + 2, NJ * NK - 1]:
    st = np.diff(d[blk])
    print("blk %3d (J %d K %d): step0 %.2f  end %.2f  median step %.3f us  steps>0.5us %d" % (
        blk, blk % NJ, blk // NJ, d[blk, 0], d[blk, -1], np.median(st), (st > 0.5).sum()))
print("blk 0 steps:", " ".join("%.2f" % x for x in d[0, :30]))
print("blk 1 steps:", " ".join("%.2f" % x for x in d[1, :30]))
print("blk 9 steps:", " ".join("%.2f" % x for x in d[NJ + 1, :30]))
# per-step phase clocks of three probe lanes of block 0 (tid 0, 64, 193)
pr = np.loadtxt(path + ".probe", dtype=np.int64)
for ps in range(3):
    r = pr[pr[:, 1] == ps][10:40]
    ph = np.diff(r[:, 2:7], axis=1)
    gap = r[1:, 2] - r[:-1, 6]
    print("probe", ps, "median cycles: crit %d shfl+x %d old %d wait %d | barrier->next %d" % (
        *np.median(ph, axis=0), np.median(gap)))
