"""Timeline of k_tile_ws from a PF_WS_TRACE dump (PF_WS_DEBUG=1 PF_WS_TRACE=<file> python bench.py ...).

    python profiles/ws_trace.py <trace.bin> [groups]

Events per tile (cycles since the CTA started; see the WS_TRACE comment in pf_tile_ws.cu): 0 builder
start, 1 builder coefficients ready, 2 builder done, 3 MMA A ready, 4+g MMA group g committed,
14 loader tile start, 15+g loader group g issued, 25+g accumulator group g ready, 35+g F group g
released, 45..49 similarity-epilogue phases. `groups` = MMA groups per tile (8 feature groups + 1
similarity group at D=1024, K=128).
"""
import sys

import numpy as np

CTAS, TILES, EV = 4, 64, 64
ng = int(sys.argv[2]) if len(sys.argv) > 2 else 9
t = np.fromfile(sys.argv[1], dtype=np.uint32).reshape(CTAS, TILES, EV).astype(np.int64)
t[t == 0xFFFFFFFF] = -1
col = lambda e: t[:, :, e]  # noqa: E731
lo, hi = 4, 60
nxt = lambda x: np.roll(x, -1, axis=1)  # noqa: E731


def med(v):
    v = v[:, lo:hi]
    return np.median(v), np.percentile(v, 90)


rows = [
    ("tile period (MMA A ready -> next A ready)", nxt(col(3)) - col(3)),
    ("builder: start -> coefficients ready", col(1) - col(0)),
    ("builder: coefficients ready -> done", col(2) - col(1)),
    ("builder done -> MMA A ready", col(3) - col(2)),
    ("MMA: A ready -> group 0 committed", col(4) - col(3)),
    ("MMA: group 0 -> last group committed", col(4 + ng - 1) - col(4)),
    ("loader: tile start -> group 0 issued", col(15) - col(14)),
    ("loader: group 0 -> last group issued", col(15 + ng - 1) - col(15)),
    ("acc: group 0 ready -> last F group released", col(35 + ng - 2) - col(25)),
    ("acc: S ready -> epilogue done", col(49) - col(25 + ng - 1)),
    ("acc:   S ready -> |F|^2 exchange", col(45) - col(25 + ng - 1)),
    ("acc:   -> pass 1 done", col(46) - col(45)),
    ("acc:   -> sums exchange", col(47) - col(46)),
    ("acc:   -> pass 2 done", col(48) - col(47)),
    ("acc:   -> epilogue done", col(49) - col(48)),
    ("acc: epilogue done -> next group 0 ready", nxt(col(25)) - col(49)),
    ("acc half 0: epilogue done -> next tile entered", nxt(col(52)) - col(49)),
    ("acc half 0: next tile entered -> waits group 0", col(50) - col(52)),
    ("acc half 0: waits group 0 -> group 0 ready", col(25) - col(50)),
    ("acc half 1: epilogue done -> next tile entered", nxt(col(53)) - col(54)),
    ("acc half 1: waits group 1 -> group 1 ready", col(26) - col(51)),
]
for name, v in rows:
    m, p = med(v)
    print(f"  {name:45s} median {m:8.0f}  p90 {p:8.0f}")

print("\nper group, cycles after the tile's MMA A-ready (median over tiles):")
print(f"  {'g':>2} {'loader issued':>14} {'MMA committed':>14} {'acc ready':>10} {'acc released':>13}")
a = col(3)
for g in range(ng):
    li = med(col(15 + g) - a)[0]
    mc = med(col(4 + g) - a)[0]
    ar = med(col(25 + g) - a)[0]
    rl = med(col(35 + g) - a)[0] if g < ng - 1 else med(col(49) - a)[0]
    print(f"  {g:2d} {li:14.0f} {mc:14.0f} {ar:10.0f} {rl:13.0f}")
