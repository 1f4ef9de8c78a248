"""Tensor-pipe rate microbenchmark (pf_bench_umma): cycles per tcgen05.mma M=128 x N x K=16."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2511_03126_b200 import _lib  # noqa: E402

out = torch.zeros(4 * 148, dtype=torch.int64, device="cuda")
reps = 2000
for n in (64, 128, 256):
    for ts in (0, 1, 2):
        for stores in (0,):
            _lib.call("pf_bench_umma", n, ts, reps, stores, out.data_ptr(), torch.cuda.current_stream().cuda_stream)
            torch.cuda.synchronize()
            o = out[: 2 * 148].view(-1, 2).double().cpu()
            per = o[:, 1].mean().item() / (reps * 8)
            ideal = 128 * n * 16 * 2 / 8192  # cycles at 8192 flop/clk/SM
            print(f"N={n:3d} {['ss', 'ts', 'ts-elect'][ts]} stores={stores}: {per:7.1f} cycles/MMA "
                  f"(issue {o[:, 0].mean().item() / (reps * 8):6.1f}); peak-rate ideal {ideal:.0f}")

# tcgen05.ld latency while the MMA stream runs (N=128, TS, elected issue)
_lib.call("pf_bench_umma", 128, 2, reps, 2, out.data_ptr(), torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
o = out[2 * 148:].view(-1, 2).double().cpu()
print(f"tcgen05.ld 32x32b.x32 + wait::ld under MMA load: {(o[:, 0] / o[:, 1].clamp(min=1)).mean().item():.1f} cycles")
