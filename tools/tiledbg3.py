"""Per-group clocks of the dataflow tile solve (EDFA_TILE_DEBUG2 dump):
t g c0(start) c1(early folded) c2(critical present) c3(end | level<<56)."""
import os, subprocess, sys
import numpy as np
path = "/tmp/tiledbg3.txt"
if len(sys.argv) < 2:
    env = dict(os.environ, EDFA_TILE_DEBUG2=path)
    subprocess.run([sys.executable, "tools/tiledbg.py"], env=env, check=True)
d = np.loadtxt(path, dtype=np.int64)
for tile in [511, 510, 438, 0]:
    r = d[d[:, 0] == tile]
    if not len(r):
        continue
    lv = r[:, 6]
    c3 = r[:, 5]
    base = r[:, 2].min()
    print("tile", tile)
    for i in np.argsort(c3):
        print("  g %2d lv %2d start %6d early %6d crit %6d end %6d" % (r[i, 1], lv[i], r[i, 2] - base, r[i, 3] - base,
                                                                    r[i, 4] - base, c3[i] - base))
