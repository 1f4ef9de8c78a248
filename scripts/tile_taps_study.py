"""Taps per tile vs tile size on a generated object (design study for the Gram tile kernel).

    python scripts/tile_taps_study.py /tmp/c5   (expects <prefix>_points.npy, _depth.npy, _meta.pkl)

Points are sorted by the 256^3 Hilbert key of csrc/pf_tile.cu (k_sort_keys); for sampled runs of
consecutive sorted points it counts, per tile size M, the exact union of the visible points' bilinear
taps (view, cell) and the box windows the prep kernel would emit (per view: the box of the visible
points' 2x2 windows, padded to an even tap count).
"""
import pickle
import sys

import numpy as np


def hilbert3(x, y, z, bits):
    X = [x.astype(np.uint32).copy(), y.astype(np.uint32).copy(), z.astype(np.uint32).copy()]
    M = np.uint32(1 << (bits - 1))
    Q = int(M)
    while Q > 1:
        P = np.uint32(Q - 1)
        for i in range(3):
            hit = (X[i] & np.uint32(Q)) != 0
            t = (X[0] ^ X[i]) & P
            X0n = np.where(hit, X[0] ^ P, X[0] ^ t)
            Xin = np.where(hit, X[i], X[i] ^ t)
            if i == 0:
                X[0] = np.where(hit, X[0] ^ P, X[0])  # i == 0: X[0]^X[0] = 0, t = 0
            else:
                X[0], X[i] = X0n, Xin
        Q >>= 1
    X[1] ^= X[0]
    X[2] ^= X[1]
    t = np.zeros_like(X[0])
    Q = int(M)
    while Q > 1:
        t ^= np.where((X[2] & np.uint32(Q)) != 0, np.uint32(Q - 1), np.uint32(0))
        Q >>= 1
    for i in range(3):
        X[i] ^= t
    key = np.zeros_like(X[0])
    for b in range(bits - 1, -1, -1):
        key = (key << np.uint32(3)) | (((X[0] >> np.uint32(b)) & 1) << 2) | (((X[1] >> np.uint32(b)) & 1) << 1) | ((X[2] >> np.uint32(b)) & 1)
    return key


def main(prefix, nsamp=300, span=4096, seed=0):
    pts = np.load(prefix + "_points.npy")
    depth = np.load(prefix + "_depth.npy")
    poses, intr, cfg = pickle.load(open(prefix + "_meta.pkl", "rb"))
    lo, hi = pts.min(0).astype(np.float64), pts.max(0).astype(np.float64)
    ext = float((hi - lo).max())
    inv = np.float32(256 / ext)
    c = np.clip(((pts - lo.astype(np.float32)) * inv).astype(np.int64), 0, 255)
    key = hilbert3(c[:, 0], c[:, 1], c[:, 2], 8)
    order = np.argsort(key, kind="stable")
    rng = np.random.default_rng(seed)
    starts = rng.integers(0, (len(pts) - span) // span, nsamp) * span
    hf, wf, d = cfg.fmap
    H = W = cfg.image
    sizes = [128, 256, 512, 1024, 2048, 4096]
    exact = {m: [] for m in sizes}
    box = {m: [] for m in sizes}
    for s in starts:
        p = pts[order[s:s + span]].astype(np.float64)
        vis = np.zeros((span, len(poses)), bool)
        tx = np.zeros((span, len(poses)), np.int64)
        ty = np.zeros((span, len(poses)), np.int64)
        dxs = np.zeros((span, len(poses)), np.int64)
        dys = np.zeros((span, len(poses)), np.int64)
        for j, pose in enumerate(poses):
            cam = p @ pose.rotation.T + pose.translation
            z = cam[:, 2]
            u = intr.fx * cam[:, 0] / z + intr.cx
            v = intr.fy * cam[:, 1] / z + intr.cy
            iu, iv = np.rint(u), np.rint(v)
            ok = (z > 0) & (iu >= 0) & (iu < W) & (iv >= 0) & (iv < H)
            iu_c = np.clip(iu, 0, W - 1).astype(np.int64)
            iv_c = np.clip(iv, 0, H - 1).astype(np.int64)
            st = depth[j][iv_c, iu_c].astype(np.float64)
            ok &= (st > 0) & (z <= st + cfg.eps)
            vis[:, j] = ok
            fu = np.clip((u + 0.5) * (wf / W) - 0.5, 0, wf - 1)
            fv = np.clip((v + 0.5) * (hf / H) - 0.5, 0, hf - 1)
            x0, y0 = np.floor(fu).astype(np.int64), np.floor(fv).astype(np.int64)
            tx[:, j], ty[:, j] = x0, y0
            dxs[:, j] = (x0 < wf - 1).astype(np.int64)
            dys[:, j] = (y0 < hf - 1).astype(np.int64)
        for m in sizes:
            for t0 in range(0, span, m):
                sl = slice(t0, t0 + m)
                taps = set()
                nbox = 0
                for j in range(len(poses)):
                    vv = vis[sl, j]
                    if not vv.any():
                        continue
                    x0, y0 = tx[sl, j][vv], ty[sl, j][vv]
                    x1, y1 = x0 + dxs[sl, j][vv], y0 + dys[sl, j][vv]
                    for a, b, c_, e in zip(x0, y0, x1, y1):
                        for yy in (b, e):
                            for xx in (a, c_):
                                taps.add((j, yy, xx))
                    w = x1.max() - x0.min() + 1
                    h = y1.max() - y0.min() + 1
                    nbox += (w * h + 1) & ~1
                exact[m].append(len(taps))
                box[m].append(nbox)
    for m in sizes:
        e, b = np.array(exact[m]), np.array(box[m])
        print(f"M={m:5d}: exact taps mean {e.mean():6.1f} p50 {np.median(e):5.0f} p99 {np.percentile(e, 99):5.0f} | "
              f"box mean {b.mean():6.1f} p50 {np.median(b):5.0f} p95 {np.percentile(b, 95):5.0f} p99 {np.percentile(b, 99):5.0f} "
              f"max {b.max():5d} | >128 {np.mean(b > 128) * 100:5.1f}% >192 {np.mean(b > 192) * 100:5.1f}% >256 {np.mean(b > 256) * 100:5.1f}%"
              f" | box/pt {b.mean() / m:6.3f}")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "/tmp/c5")
