"""Timeline of k_tile_ws from a PF_WS_TRACE dump (PF_WS_DEBUG=1 PF_WS_TRACE=<file> python bench.py ...).

    python profiles/ws_trace.py <trace.bin> [ngroups]

Events per tile (cycles since the CTA started): 0 build start, 1 build zeroed, 2 build done,
3 mma A ready, 4.. mma group g issued, 13 loader tile start, 14.. loader group g published,
23.. accumulator group g ready (the last group is the similarity group).
"""
import sys

import numpy as np

CTAS, TILES = 4, 64
t = np.fromfile(sys.argv[1], dtype=np.uint32).reshape(CTAS, TILES, 32).astype(np.int64)
ng = int(sys.argv[2]) if len(sys.argv) > 2 else 9
t[t == 0xFFFFFFFF] = -1


def col(e):
    return t[:, :, e]


lo, hi = 4, 60  # steady-state tiles
period = np.diff(col(3), axis=1)[:, lo:hi]
print(f"tile period (mma A-ready to A-ready): median {np.median(period):.0f} cycles")
rows = [
    ("build: start -> zeroed", col(1) - col(0)),
    ("build: zeroed -> done", col(2) - col(1)),
    ("build done(t+1) - mma A ready(t)", np.roll(col(2), -1, axis=1) - col(3)),
    ("mma: A ready -> last group issued", col(4 + ng - 1) - col(3)),
    ("mma: last issued(t) -> A ready(t+1)", np.roll(col(3), -1, axis=1) - col(4 + ng - 1)),
    ("loader: tile start -> last group published", col(14 + ng - 1) - col(13)),
    ("loader: group published -> mma issued (mean over groups)",
     np.mean([col(4 + g) - col(14 + g) for g in range(ng)], axis=0)),
    ("acc: mma last issued -> S ready", col(23 + ng - 1) - col(4 + ng - 1)),
    ("acc: group g ready - mma group g issued (mean)", np.mean([col(23 + g) - col(4 + g) for g in range(ng)], axis=0)),
]
for name, v in rows:
    v = v[:, lo:hi]
    print(f"  {name:58s} median {np.median(v):8.0f}  p90 {np.percentile(v, 90):8.0f}")
c = 0
base = t[c, 10, 3]
print(f"CTA {c} tiles 10-12, cycles relative to tile 10 A-ready:")
for tl in range(10, 13):
    r = t[c, tl] - base
    print(f" tile {tl}: build {r[0]}..{r[1]}..{r[2]}  mmaA {r[3]}  mma groups {list(r[4:4 + ng])}")
    print(f"          loader start {r[13]} published {list(r[14:14 + ng])}")
    print(f"          acc ready {list(r[23:23 + ng])}")
