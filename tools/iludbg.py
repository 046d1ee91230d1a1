"""Row timeline of the sync-free ILU(0) factorisation (EDFA_ILU_DEBUG dump):
per wavefront level (i+j+k), claim / pivots-ready / done times."""
import os, subprocess, sys
import numpy as np
path = "/tmp/ilu_dbg.bin"
if len(sys.argv) < 2:
    env = dict(os.environ, EDFA_ILU_DEBUG=path)
    subprocess.run([sys.executable, "tools/tiledbg.py"], env=env, check=True)
d = np.fromfile(path, dtype=np.int64).reshape(-1, 3)
t0 = d[:, 0].min()
d = (d - t0) / 1e3
n = d.shape[0]
nx = round(n ** (1 / 3))
e = np.arange(n)
lev = e % nx + (e // nx) % nx + e // (nx * nx)
print("span us %.1f  median row time (claim->done) %.2f us  wait (claim->pivots) %.2f  work (pivots->done) %.2f" % (
    d[:, 2].max(), np.median(d[:, 2] - d[:, 0]), np.median(d[:, 1] - d[:, 0]), np.median(d[:, 2] - d[:, 1])))
for L in [0, 1, 2, 10, 50, 95, 100, 150, 189]:
    m = lev == L
    print("lev %3d rows %4d claim %.1f-%.1f  ready %.1f-%.1f  done %.1f-%.1f" % (
        L, m.sum(), d[m, 0].min(), d[m, 0].max(), d[m, 1].min(), d[m, 1].max(), d[m, 2].min(), d[m, 2].max()))
