"""Timeline of k_tile_ws from a PF_WS_TRACE dump (PF_WS_DEBUG=1 PF_WS_TRACE=<file> python bench.py ...).

    python profiles/ws_trace.py <trace.bin>

Events per tile (cycles since the CTA started): 0 builder start, 1 builder coefficients ready,
2 builder done, 3 MMA A ready, 4 / 5 / 6 MMA first / middle / last group issued, 13 loader tile
start, 14 / 15 loader first / last chunk issued, 23 / 24 accumulator first / last feature group
ready, 25 similarity group ready, 26 accumulator epilogue done (slot released).
"""
import sys

import numpy as np

CTAS, TILES = 4, 64
t = np.fromfile(sys.argv[1], dtype=np.uint32).reshape(CTAS, TILES, 32).astype(np.int64)
t[t == 0xFFFFFFFF] = -1
col = lambda e: t[:, :, e]  # noqa: E731
lo, hi = 4, 60
nxt = lambda x: np.roll(x, -1, axis=1)  # noqa: E731
rows = [
    ("tile period (MMA A ready -> next A ready)", nxt(col(3)) - col(3)),
    ("builder: start -> done", col(2) - col(0)),
    ("MMA: A ready -> first group issued", col(4) - col(3)),
    ("MMA: first -> middle group issued", col(5) - col(4)),
    ("MMA: middle -> last group issued", col(6) - col(5)),
    ("MMA: last issued -> next A ready", nxt(col(3)) - col(6)),
    ("loader: first -> last chunk issued", col(15) - col(14)),
    ("acc: MMA first issued -> first F ready", col(23) - col(4)),
    ("acc: first F -> last F ready", col(24) - col(23)),
    ("acc: MMA last issued -> S ready", col(25) - col(6)),
    ("acc: S ready -> epilogue done", col(26) - col(25)),
    ("acc:   S ready -> after |F|^2 exchange barrier", col(27) - col(25)),
    ("acc:   barrier -> pass 1 done (+ stash)", col(28) - col(27)),
    ("acc:   pass 1 -> after sums exchange barrier", col(29) - col(28)),
    ("acc:   barrier -> pass 2 done", col(30) - col(29)),
    ("acc:   pass 2 -> props / atomics / release", col(26) - col(30)),
    ("acc: epilogue done -> next first F ready", nxt(col(23)) - col(26)),
]
for name, v in rows:
    v = v[:, lo:hi]
    print(f"  {name:45s} median {np.median(v):8.0f}  p90 {np.percentile(v, 90):8.0f}")
