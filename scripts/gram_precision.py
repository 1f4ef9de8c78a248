"""Precision of the Gram formulation of |F| (design study for csrc/pf_gram.cu).

    python scripts/gram_precision.py random|corr      (needs /tmp/c5_{points,depth}.npy, /tmp/c5_meta.pkl
                                                       from workloads.generate("c5"), see tile_taps_study.py)

For sampled 512-point Hilbert tiles of a C5 object: the exact |F|^2 = |W T|^2 (W = bf16 bilinear weights,
T = the tiles tap rows from bf16 maps) against w^T bf16(T T^T) w (the kernel: Gram rounded to bf16 as the
MMA B operand), and the resulting similarity / softmax-weight differences. "corr" uses strongly
correlated feature cells and text aligned with them (large similarities), the worst case for the
rounding of the Gram entries.
"""
import numpy as np, pickle, sys
sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/scripts')
from tile_taps_study import hilbert3
from paper_2511_03126_b200.workloads import f32_to_bf16_bits, bf16_bits_to_f32
pts = np.load('/tmp/c5_points.npy'); depth = np.load('/tmp/c5_depth.npy')
poses, intr, cfg = pickle.load(open('/tmp/c5_meta.pkl','rb'))
hf, wf, d = cfg.fmap; H=W=cfg.image; V=len(poses)
rng = np.random.default_rng(1)
def bf(x): return bf16_bits_to_f32(f32_to_bf16_bits(np.asarray(x, np.float32))).astype(np.float64)
mode = sys.argv[1]
if mode == 'random':
    fm = rng.standard_normal((V, hf, wf, d), dtype=np.float32)
else:  # correlated: shared base vector + small per-cell noise (cosines ~0.9 between cells)
    base = rng.standard_normal(d, dtype=np.float32)
    fm = base + 0.35 * rng.standard_normal((V, hf, wf, d), dtype=np.float32)
fm /= np.linalg.norm(fm, axis=3, keepdims=True)
fm = bf(fm).reshape(V * hf * wf, d)
text = rng.standard_normal((128, d)); text /= np.linalg.norm(text, axis=1, keepdims=True)
if mode != 'random':  # text aligned with the base: large similarities
    text = text * 0.3 + base / np.linalg.norm(base); text /= np.linalg.norm(text, axis=1, keepdims=True)
G = fm @ text.T
lo, hi = pts.min(0).astype(np.float64), pts.max(0).astype(np.float64)
inv = np.float32(256 / float((hi - lo).max()))
c = np.clip(((pts - lo.astype(np.float32)) * inv).astype(np.int64), 0, 255)
order = np.argsort(hilbert3(c[:, 0], c[:, 1], c[:, 2], 8), kind='stable')
M_T = 512
errs_F, errs_Fd, errs_s, errs_w = [], [], [], []
for s0 in rng.integers(0, len(pts) // M_T - 1, 60) * M_T:
    p = pts[order[s0:s0 + M_T]].astype(np.float64)
    rows, cols, vals = [], [], []
    for j, pose in enumerate(poses):
        cam = p @ pose.rotation.T + pose.translation; z = cam[:, 2]
        u = intr.fx * cam[:, 0] / z + intr.cx; v = intr.fy * cam[:, 1] / z + intr.cy
        iu, iv = np.rint(u), np.rint(v)
        ok = (z > 0) & (iu >= 0) & (iu < W) & (iv >= 0) & (iv < H)
        st = depth[j][np.clip(iv,0,H-1).astype(int), np.clip(iu,0,W-1).astype(int)]
        ok &= (st > 0) & (z <= st + cfg.eps)
        fu = np.clip((u + 0.5) * (wf / W) - 0.5, 0, wf - 1); fv = np.clip((v + 0.5) * (hf / H) - 0.5, 0, hf - 1)
        x0 = np.floor(fu).astype(int); y0 = np.floor(fv).astype(int)
        x1 = np.minimum(x0 + 1, wf - 1); y1 = np.minimum(y0 + 1, hf - 1)
        wx = fu - x0; wy = fv - y0
        for yy, xx, ww in ((y0, x0, (1-wy)*(1-wx)), (y0, x1, (1-wy)*wx), (y1, x0, wy*(1-wx)), (y1, x1, wy*wx)):
            r = np.nonzero(ok)[0]
            rows.append(r); cols.append(j * hf * wf + yy[r] * wf + xx[r]); vals.append(ww[r])
    rows = np.concatenate(rows); cols = np.concatenate(cols); vals = np.concatenate(vals)
    taps, cidx = np.unique(cols, return_inverse=True)
    Wm = np.zeros((M_T, len(taps)))
    np.add.at(Wm, (rows, cidx), vals)
    Wb = bf(Wm)
    T = fm[taps]
    F = Wb @ T
    nF2 = (F ** 2).sum(1)
    Mx = T @ T.T
    Mb = bf(Mx)
    nF2_g = np.einsum('rt,rt->r', Wb, Wb @ Mb)
    dg = np.diag(Mx) - np.diag(Mb)
    nF2_gd = nF2_g + (Wb ** 2) @ dg
    ok = nF2 > 0
    errs_F.append(np.abs(np.sqrt(nF2_g[ok]) / np.sqrt(nF2[ok]) - 1))
    errs_Fd.append(np.abs(np.sqrt(nF2_gd[ok]) / np.sqrt(nF2[ok]) - 1))
    S = Wb @ bf(G[taps])
    s_ref = S[ok] / np.sqrt(nF2[ok])[:, None]; s_g = S[ok] / np.sqrt(nF2_gd[ok])[:, None]
    errs_s.append(np.abs(s_g - s_ref).max(1))
    def sm(x):
        x = x / 0.1; x -= x.max(1, keepdims=True); e = np.exp(x); return e / e.sum(1, keepdims=True)
    errs_w.append(np.abs(sm(s_g) / sm(s_ref) - 1).max(1))
for nm, e in (('|F| rel (bf16 M)', errs_F), ('|F| rel (+diag fix)', errs_Fd), ('max|ds|', errs_s), ('weights rel', errs_w)):
    e = np.concatenate(e); print(f"{mode} {nm}: mean {e.mean():.2e} p99 {np.percentile(e, 99):.2e} max {e.max():.2e}")
