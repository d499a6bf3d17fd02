"""tools/mgaq_kernels.py -- the three MGAQ kernel kinds on ONE cfg2 tensor of
8192 x 11008 bf16 (90,177,536 elements: silu.in / down.in size), for an
`ncu --set full` capture whose per-element figures are then exact:
quant_group_kernel (per-group 1x16), group_amax_kernel (Group Scaling stage 1+2)
and quant_tensor_kernel (per-tensor encode)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2410_19313_b200 import coatsim as coat
    g = torch.Generator(device="cuda").manual_seed(9)
    x = (torch.randn(8192, 11008, device="cuda", generator=g) * 2).to(torch.bfloat16)
    x[::100] *= 50
    for _ in range(2):
        coat.quantize(x, coat.QuantGeometry.per_group(16))
        coat.quantize(x, coat.QuantGeometry.per_tensor())
    torch.cuda.synchronize()
    print("mgaq kernels ok")


if __name__ == "__main__":
    main()
