"""Per-tile timeline of one ILU L-solve (EDFA_TILE_DEBUG dump), pipelined kernel.
dbg columns: t, start, first-level start, levels end, tile end, -, cycles/step"""
import os, subprocess, sys
import numpy as np
path = "/tmp/tiledbg.txt"
if len(sys.argv) < 2:
    env = dict(os.environ, EDFA_TILE_DEBUG=path)
    subprocess.run([sys.executable, "tools/tiledbg.py"], env=env, check=True)
d = np.loadtxt(path, dtype=np.int64)
t0 = d[:, 1].min()
st, fl, le, te, cyc = (d[:, 1] - t0) / 1e3, (d[:, 2] - t0) / 1e3, (d[:, 3] - t0) / 1e3, (d[:, 4] - t0) / 1e3, d[:, 6]
print("span us", te.max())
print("median: wait-before-first-level us %.2f  levels us %.2f  tail us %.2f  cyc/step %d" % (
    np.median(fl - st), np.median(le - fl), np.median(te - le), np.median(cyc)))
# tile grid 8x8x8 tiles, natural order: print finish time along the diagonal
NX = 8
for k in range(8):
    t = k + NX * (k + NX * k)
    print("diag tile", t, "start %.1f first %.1f levels_end %.1f end %.1f" % (st[t], fl[t], le[t], te[t]))
for t in [0, 1, 2, 3, 8, 64]:
    print("tile", t, "start %.1f first %.1f levels_end %.1f end %.1f cyc %d" % (st[t], fl[t], le[t], te[t], cyc[t]))
print("chain (reverse solve):")
for t in [511, 510, 503, 447, 502, 439, 446, 438, 437, 430, 374, 365]:
    print("tile", t, "start %.1f first %.1f levels_end %.1f end %.1f" % (st[t], fl[t], le[t], te[t]))
