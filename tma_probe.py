import torch, sys
sys.path.insert(0, '.')
from paper_2511_03126_b200 import _lib
src = torch.arange(6*6*64, dtype=torch.float32, device='cuda').reshape(6, 6, 64).to(torch.bfloat16)
for row_off in [0, 3, 5, 8, 13]:
    for (bw, bh) in [(2, 2), (3, 2), (4, 4)]:
        out = torch.empty(bw*bh, 64, dtype=torch.bfloat16, device='cuda')
        try:
            _lib.call("pf_selftest_tma", src.data_ptr(), 6, 6, 1, 1, bw, bh, row_off, out.data_ptr(), torch.cuda.current_stream().cuda_stream)
            torch.cuda.synchronize()
        except Exception as e:
            print("row_off", row_off, bw, bh, "ERROR", str(e)[:100]); sys.exit(0)
        ref = src[1:1+bh, 1:1+bw].reshape(-1, 64)
        print("row_off", row_off, "box", bw, bh, "match", bool(torch.equal(out, ref)))
