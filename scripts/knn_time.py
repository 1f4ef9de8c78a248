"""Device characteristic_length (k-NN, integrate.py:72-95) timing on a workload's points."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2511_03126_b200 as pf  # noqa: E402
from paper_2511_03126_b200 import _lib, workloads  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
wl = workloads.generate(name, device_splat=True)
p = torch.from_numpy(wl.points).cuda()
n = p.shape[0]
ws = torch.empty(int(_lib.load().pf_knn_workspace_bytes(n)), dtype=torch.uint8, device="cuda")
out = torch.zeros(1, dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream().cuda_stream
for _ in range(2):
    _lib.call("pf_knn_kth_distance", p.data_ptr(), n, 8, out.data_ptr(), None, ws.data_ptr(), st)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
reps = 5
for _ in range(reps):
    _lib.call("pf_knn_kth_distance", p.data_ptr(), n, 8, out.data_ptr(), None, ws.data_ptr(), st)
b.record()
torch.cuda.synchronize()
L = float(np.sqrt(np.pi / 8 * out.item()))
print(f"{name}: N={n} characteristic_length={L:.6f} m, device k-NN {a.elapsed_time(b) / reps:.3f} ms")
if n <= 3_000_000:
    from oracle import propfield_oracle as O

    t0 = time.perf_counter()
    Lr = O.characteristic_length(wl.points.astype(np.float64))
    print(f"  cKDTree oracle: {Lr:.6f} m in {time.perf_counter() - t0:.2f} s (rel diff {abs(L - Lr) / Lr:.2e})")
