import os, sys, numpy as np, torch
os.environ["PF_WS_DEBUG"] = "1"
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
for _ in range(2):
    a = pf.fuse_and_query(pts, views, tables, grid=wl.cfg.grid)
torch.cuda.synchronize()
