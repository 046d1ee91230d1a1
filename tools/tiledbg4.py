"""Cross-tile hand-off timeline of the dataflow tile solve (EDFA_TILE_DEBUG2,
globaltimer stamps): per level, when the upstream tile finished it and when the
downstream tile's groups got their early dependencies / critical ones."""
import os, subprocess, sys
import numpy as np
path = "/tmp/tiledbg4.txt"
if len(sys.argv) < 2:
    env = dict(os.environ, EDFA_TILE_DEBUG2=path)
    subprocess.run([sys.executable, "tools/tiledbg.py"], env=env, check=True)
d = np.loadtxt(path, dtype=np.int64)
t0 = d[:, 2].min()
def per_level(tile):
    r = d[d[:, 0] == tile]
    lv = r[:, 6]
    c3 = r[:, 5] - t0
    out = {}
    for L in np.unique(lv):
        m = lv == L
        out[int(L)] = ((r[m, 2] - t0).min(), (r[m, 3] - t0).max(), (r[m, 4] - t0).max(), c3[m].max())
    return out
for chain in ([511, 510, 509, 508], [511, 503, 495], [511, 447, 383]):
    print("chain", chain)
    for L in range(22):
        row = []
        for t in chain:
            pl = per_level(t)
            if L in pl:
                s, e, c, f = pl[L]
                row.append("%6.2f/%6.2f/%6.2f/%6.2f" % (s / 1e3, e / 1e3, c / 1e3, f / 1e3))
        print("  lv %2d  " % L + "   ".join(row))
