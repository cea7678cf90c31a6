"""Summarise a trace_prefill.py JSON dump: per event kind, the median interval between successive
events in the steady state, and per position the latencies K issue -> K landed (ev 0 -> 15) and
V issue -> V landed (ev 1 -> 14), V landed -> PV issue (14 -> 3), plus the first/last times."""
import json
import sys

import numpy as np

d = json.load(open(sys.argv[1]))
ev = {int(k): np.array([x for x in v if x is not None], dtype=np.float64) for k, v in d["events"].items()}
names = {0: "K issue", 1: "V issue", 2: "S issue", 3: "PV issue", 5: "WG0 S-ready", 6: "WG0 P-ready",
         7: "WG1 S-ready", 8: "WG1 P-ready", 10: "sched publish", 14: "V landed", 15: "K landed"}
print("total cycles", d["total"])
for k, nm in names.items():
    a = ev.get(k)
    if a is None or len(a) < 8:
        continue
    di = np.diff(a)
    lo, hi = len(di) // 4, 3 * len(di) // 4
    print(f"{nm:14s} n={len(a):4d} first {a[0]:9.0f} last {a[-1]:9.0f} median interval {np.median(di[lo:hi]):7.0f}")


def lat(a, b, nm):
    if a in ev and b in ev:
        n = min(len(ev[a]), len(ev[b]))
        x = ev[b][:n] - ev[a][:n]
        print(f"{nm:24s} median {np.median(x[n // 4: 3 * n // 4]):7.0f}  p90 {np.percentile(x, 90):7.0f}")


lat(0, 15, "K issue -> landed")
lat(1, 14, "V issue -> landed")
lat(14, 3, "V landed -> PV issue")
lat(5, 6, "WG0 S-ready -> P-ready")
lat(7, 8, "WG1 S-ready -> P-ready")
