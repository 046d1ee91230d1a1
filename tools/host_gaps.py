"""Host scheduling hiccups: longest perf_counter gaps of a busy loop."""
import sys, time
dur = float(sys.argv[1]) if len(sys.argv) > 1 else 10.0
t_end = time.perf_counter() + dur
last = time.perf_counter()
gaps = []
while True:
    t = time.perf_counter()
    if t - last > 0.002:
        gaps.append(round((t - last) * 1e3, 1))
    last = t
    if t > t_end:
        break
print("gaps>2ms:", len(gaps), "max", max(gaps) if gaps else 0, sorted(gaps)[-10:])
