"""tools/gemm_vs_library.py -- K4's BF16 dgrad and FP8 forward next to the
library kernels on the same cfg4 shapes (cuBLAS dY . W^T, cuBLASLt
torch._scaled_mm), one launch each after warm-up, for an ncu capture that
names the library kernels (tile / cluster shape) and compares their metrics."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2410_19313_b200 import coatsim as coat
    M, K, N = 8192, 5120, 13824
    g = torch.Generator(device="cuda").manual_seed(11)
    x = (torch.randn(M, K, device="cuda", generator=g)).to(torch.bfloat16)
    w = torch.randn(K, N, device="cuda", generator=g) / K ** 0.5
    qx = coat.quantize(x, coat.QuantGeometry.per_tensor())
    qw = coat.quantize(w, coat.QuantGeometry.per_tensor())
    dy = (torch.randn(M, N, device="cuda", generator=g) * 1e-3).to(torch.bfloat16)
    wd = w.to(torch.bfloat16)
    a = qx.codes.view(torch.float8_e4m3fn)
    wt = qw.codes.t().contiguous().view(torch.float8_e4m3fn)
    one = torch.ones((), device="cuda")
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("cmp")
    coat.linear_dgrad(dy, qw)
    torch.matmul(dy, wd.t())
    coat.fp8_linear(qx, qw)
    torch._scaled_mm(a, wt.t(), scale_a=one, scale_b=one, out_dtype=torch.float32)
    torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
