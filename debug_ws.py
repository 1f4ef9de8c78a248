import os, sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2511_03126_b200 as pf
from paper_2511_03126_b200 import workloads
wl = workloads.generate("c5", device_splat=True)
nv = wl.cfg.nviews
R = np.stack([p.rotation for p in wl.poses]); tv = np.stack([p.translation for p in wl.poses])
intr = np.tile([wl.intrinsics.fx, wl.intrinsics.fy, wl.intrinsics.cx, wl.intrinsics.cy], (nv, 1))
fmap = torch.from_numpy(wl.fmaps.view(np.int16)).cuda().view(torch.bfloat16)
views = pf.ViewSet.from_tensors(R, tv, intr, wl.depth.cuda(), fmap)
tables = pf.QueryTables.build(wl.text, wl.values, wl.mid_theta)
pts = torch.from_numpy(wl.points).cuda()
a = pf.fuse_and_query(pts, views, tables, grid=wl.cfg.grid, write_sims=True)
sa, pa = a.sims.clone(), a.props.clone()
b = pf.fuse_and_query(pts, views, tables, grid=wl.cfg.grid, write_sims=True, force_simt=True)
sb, pb = b.sims, b.props
rel = ((pa[:, 0] - pb[:, 0]).abs() / pb[:, 0].abs().clamp_min(1e-30))
bad = torch.nonzero(rel > 1e-2).flatten()
print("bad points", bad.numel(), "max rel", float(rel.max()))
ds = (sa - sb).abs().max(dim=1).values
print("sims maxdiff quantiles", [float(torch.quantile(ds[:1000000], q)) for q in (0.5, 0.99, 0.9999)], float(ds.max()))
badS = torch.nonzero(ds > 1e-3).flatten()
print("bad sims rows", badS.numel())
for i in badS[:8].tolist():
    r = (sa[i] / sb[i]).cpu().numpy()
    print(i, "counts", int(b.counts[i]), "ratio sa/sb first 6", np.round(r[:6], 4), "sa", np.round(sa[i,:4].cpu().numpy(),4), "sb", np.round(sb[i,:4].cpu().numpy(), 4))
