"""Fused producers + MGAQ vs the oracle and the
reference's own decoder-layer tape.

RMSNorm block: bit-exact (row sums in the reference's sequential order).
SiLU*mul block: every quantizer bit-exact given its fp32 input; silu itself
uses CUDA's expf (<= 2 ulp) where the reference uses glibc's -> the share of
mul.in.silu codes that differ from the reference is measured and bounded.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _np(t):
    import torch
    return (t.float() if t.dtype == torch.bfloat16 else t).cpu().numpy()


def _bf16(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(torch.bfloat16)


@pytest.mark.parametrize("rows,h,dtype", [(96, 4096, "bf16"), (33, 512, "fp32"), (8, 11008, "bf16"),
                                          (89, 272, "bf16"), (7, 16, "fp32"),   # odd groups per row
                                          (8192, 4096, "bf16")])   # the last: cfg2's full rmsnorm input
def test_rmsnorm_block_bit_exact_vs_oracle(coat, port, rows, h, dtype):
    import torch
    x = port.generate(1, (rows, h), 0.05, 30.0, 11)
    if dtype == "bf16":
        xt = _bf16(x).cuda()
        x = xt.float().cpu().numpy()
    else:
        xt = torch.from_numpy(x).cuda()
    w = (1.0 + 0.1 * port.generate(0, (h,), 0.0, 1.0, 12)).astype(np.float32)
    qx, qy, rms, y = coat.rmsnorm_quantize(xt, torch.from_numpy(w), eps=1e-6, return_y=True)
    xc, xs = port.quantize(x, 16)
    assert np.array_equal(_np(qx.codes), xc) and np.array_equal(_np(qx.scales), xs)
    y_ref = port.rmsnorm(port.dequantize(xc, xs, 16), w, 1e-6)
    assert np.array_equal(_np(y).view(np.uint32), y_ref.view(np.uint32))
    yc, ys = port.quantize(y_ref, 0)
    assert np.array_equal(_np(qy.codes), yc) and np.array_equal(_np(qy.scales), ys)


def test_rmsnorm_block_matches_reference_layer_tape(coat, ref):
    import torch
    H, I, heads, S, B = 64, 128, 4, 32, 2
    x = ref.generate(1, (B * S, H), 0.05, 20.0, 3)
    c_in, s_in, _, rms1, _ = ref.layer_tape(x, "rmsnorm1.in", H, I, heads, S, B)
    c_q, s_q, _, _, _ = ref.layer_tape(x, "qkv.in", H, I, heads, S, B)
    qx, qy, _ = coat.rmsnorm_quantize(torch.from_numpy(x).cuda(), torch.from_numpy(rms1), eps=1e-6)
    assert np.array_equal(_np(qx.codes).reshape(-1), c_in) and np.array_equal(_np(qx.scales), s_in)
    assert np.array_equal(_np(qy.codes).reshape(-1), c_q) and np.array_equal(_np(qy.scales), s_q)


@pytest.mark.parametrize("rows,cols", [(64, 11008), (40, 512), (37, 272), (8192, 11008)])   # the last: cfg2
def test_silu_mul_block(coat, port, rows, cols):
    import torch
    g = _bf16(port.generate(1, (rows, cols), 0.02, 8.0, 21) * np.float32(2.0))
    u = _bf16(port.generate(1, (rows, cols), 0.02, 8.0, 22))
    qg, qs, qu, qp, prod = coat.silu_mul_quantize(g.cuda(), u.cuda(), return_prod=True)
    gn, un = g.float().numpy(), u.float().numpy()
    gc, gs = port.quantize(gn, 16)
    uc, us = port.quantize(un, 16)
    assert np.array_equal(_np(qg.codes), gc) and np.array_equal(_np(qg.scales), gs)
    assert np.array_equal(_np(qu.codes), uc) and np.array_equal(_np(qu.scales), us)
    # the product and its per-tensor quantization are exact given the GPU's silu codes
    s_dq = port.dequantize(_np(qs.codes), _np(qs.scales), 16)
    p_ref = (s_dq * port.dequantize(uc, us, 16)).astype(np.float32)
    assert np.array_equal(_np(prod).view(np.uint32), p_ref.view(np.uint32))
    pc, ps = port.quantize(p_ref, 0)
    assert np.array_equal(_np(qp.codes), pc) and np.array_equal(_np(qp.scales), ps)
    # silu: CUDA expf vs glibc expf -> a tiny share of mul.in.silu codes may differ
    sc, ss = port.quantize(port.silu(port.dequantize(gc, gs, 16)), 16)
    diff = np.count_nonzero(_np(qs.codes) != sc) / sc.size
    assert diff < 1e-3, diff


def test_rmsnorm_block_signed_zeros(coat, port):
    """x values that quantize to -0 (code 0x80: a tiny negative next to a large
    group max) give x_used = -0 and rmsnorm -0 / rms * w = -0 (flow.cpp:56-71);
    the division's fast path must keep the sign (found at cfg2's full size)."""
    import torch
    rows, h = 16, 256
    x = port.generate(1, (rows, h), 0.0, 1.0, 31)
    x[:, ::16] = 300.0                       # each 1x16 group's max
    x[:, 1::16] = -1e-6                      # -> code 0x80 after quantization
    x[:, 2::16] = 1e-6                       # -> code 0x00
    xt = _bf16(x).cuda()
    x = xt.float().cpu().numpy()
    w = np.linspace(0.5, 1.5, h).astype(np.float32)
    w[5::7] *= -1.0                          # negative weights flip the zero's sign
    qx, qy, rms, y = coat.rmsnorm_quantize(xt, torch.from_numpy(w), eps=1e-6, return_y=True)
    xc, xs = port.quantize(x, 16)
    assert (xc == 0x80).any()
    y_ref = port.rmsnorm(port.dequantize(xc, xs, 16), w, 1e-6)
    assert np.array_equal(_np(y).view(np.uint32), y_ref.view(np.uint32))
    yc, ys = port.quantize(y_ref, 0)
    assert np.array_equal(_np(qy.codes), yc) and np.array_equal(_np(qy.scales), ys)
