"""tools/gemm_kernels.py -- K4 on the cfg4 shapes, one launch per epilogue kind,
for an `ncu --set full` capture: the FP8 forward with fp32 output, the same
forward with the per-group 1x16 quantizing epilogue, and the fused gate/up +
SiLU*mul GEMM (x 8192 x 5120, W 5120 x 13824; the cfg4 weight as both gate and
up), then the BF16 dgrad and wgrad."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2410_19313_b200 import coatsim as coat
    M, K, N = 8192, 5120, 13824
    g = torch.Generator(device="cuda").manual_seed(11)
    x = (torch.randn(M, K, device="cuda", generator=g)).to(torch.bfloat16)
    x[::100] *= 50
    w = torch.randn(K, N, device="cuda", generator=g) / K ** 0.5
    qx = coat.quantize(x, coat.QuantGeometry.per_tensor())
    qw = coat.quantize(w, coat.QuantGeometry.per_tensor())
    dy = (torch.randn(M, N, device="cuda", generator=g) * 1e-3).to(torch.bfloat16)
    coat.fp8_linear(qx, qw)
    coat.fp8_linear_q16(qx, qw)
    coat.fp8_upgate_silu(qx, qw, qw)
    coat.linear_dgrad(dy, qw)
    coat.linear_wgrad(qx, dy)
    torch.cuda.synchronize()
    print("gemm kernels ok")


if __name__ == "__main__":
    main()
