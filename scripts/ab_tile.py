"""A/B the tile-path stage times of two builds of the library on the same box:
    python scripts/ab_tile.py <lib_a.so> <lib_b.so> [more.so ...] [config]
Each library runs in its own process (reduce=False: no voxel-mass finalisation)."""
import json
import os
import subprocess
import sys

if len(sys.argv) > 1 and sys.argv[1] == "--child":
    lib_path, cfg_name = sys.argv[2], sys.argv[3]
    sys.path.insert(0, ".")
    import ctypes as C

    import numpy as np
    import torch

    from paper_2511_03126_b200 import _lib

    probe = C.CDLL(lib_path)
    for name in list(_lib.SIGNATURES):
        if not hasattr(probe, name):
            del _lib.SIGNATURES[name]
    _lib.load(lib_path)
    import paper_2511_03126_b200 as pf
    from paper_2511_03126_b200 import workloads

    wl = workloads.generate(cfg_name, device_splat=True)
    cfg = wl.cfg
    nv = cfg.nviews
    R = np.stack([p.rotation for p in wl.poses])
    tv = np.stack([p.translation for p in wl.poses])
    intr = np.tile([wl.intrinsics.fx, wl.intrinsics.fy, wl.intrinsics.cx, wl.intrinsics.cy], (nv, 1))
    fm = torch.from_numpy(wl.fmaps.view(np.int16)).cuda().view(torch.bfloat16)
    views = pf.ViewSet.from_tensors(R, tv, intr, wl.depth.cuda(), fm)
    tables = pf.QueryTables.build(wl.text, wl.values, wl.mid_theta)
    pts = torch.from_numpy(wl.points).cuda()
    bufs = pf.FuseBuffers(pts.shape[0], views, tables, cfg.grid)
    for _ in range(3):
        pf.fuse_and_query(pts, views, tables, grid=cfg.grid, buffers=bufs, reduce=False)
    torch.cuda.synchronize()
    _lib.stage_timing(True)
    for _ in range(8):
        bufs.grid_partials.zero_()
        pf.fuse_and_query(pts, views, tables, grid=cfg.grid, buffers=bufs, reduce=False)
    torch.cuda.synchronize()
    n, st = _lib.stage_times()
    print(json.dumps({k: v / n for k, v in st.items()}))
else:
    libs = [a for a in sys.argv[1:] if a.endswith(".so")]
    rest = [a for a in sys.argv[1:] if not a.endswith(".so")]
    cfg = rest[0] if rest else "c5"
    for rep in range(2):
        for lib in libs:
            out = subprocess.run([sys.executable, __file__, "--child", lib, cfg], capture_output=True, text=True)
            line = [x for x in out.stdout.splitlines() if x.startswith("{")]
            print(os.path.basename(lib), line[-1] if line else out.stderr[-500:], flush=True)
