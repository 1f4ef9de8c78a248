"""Loader microbenchmark (pf_bench_gather): bytes/clk/SM of cp.async vs TMA gather4 row gathers."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2511_03126_b200 import _lib  # noqa: E402

cells = 87616
src = torch.randn(cells, 1024, device="cuda").to(torch.bfloat16)
out = torch.zeros(148, dtype=torch.int64, device="cuda")
stages = 2000
for mode in (0, 1, 2, 0, 1, 2):
    _lib.call("pf_bench_gather", src.data_ptr(), cells, stages, mode, out.data_ptr(),
              torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    cyc = out.double().mean().item()
    print(f"{['cp.async', 'tma gather4', 'gather4 x4'][mode]:12s}: {stages * 16384 / cyc:6.1f} B/clk/SM "
          f"({stages * 16384 * 148 / cyc * 1.9e9 / 1e12:.2f} TB/s at 1.9 GHz)")
