"""GPU parity: the per-tensor FP8 linear (K4, tcgen05/TMEM/TMA) and its BF16
backward GEMMs.

Reference: flow.cpp:21-33 (matmul, sequential fp32 accumulation), 36-46
(matmul_nt), 548-552/636-637 (call sites), 360-395 (transposed FP8 codes).
Tolerance: |y - y_ref| <= tau * sum_p |a_ip b_pj|; E4M3 x
E4M3 products are exact in fp32, so the only differences are accumulation
order/precision.  tau is stated per test and the measured value printed.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TAU = 2.0 ** -16   # fp32 accumulation over K <= 5120 terms, order-independent bound


def _quant_pair(coat, M, K, N, seed):
    import torch
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.randn(M, K, device="cuda", generator=g)
    x[:: 37] *= 50.0                           # outlier token rows (ActivationWithOutliers)
    w = torch.randn(K, N, device="cuda", generator=g) / K ** 0.5
    qx = coat.quantize(x.to(torch.bfloat16), coat.QuantGeometry.per_tensor())
    qw = coat.quantize(w, coat.QuantGeometry.per_tensor())
    return qx, qw


def _ratio(y, ref, bound):
    import torch
    err = (y.double() - ref).abs()
    return float((err / bound.clamp_min(1e-300)).max())


@pytest.mark.parametrize("M,K,N", [(16, 32, 16), (128, 256, 256), (200, 272, 400), (512, 1024, 768), (600, 512, 768),
                                   (384, 5120, 13824), (8192, 5120, 13824)])   # the last: cfg4 at full size
def test_fp8_linear_forward(coat, M, K, N):
    import torch
    qx, qw = _quant_pair(coat, M, K, N, seed=M + N)
    y = coat.fp8_linear(qx, qw)
    torch.cuda.synchronize()
    a = coat.decode_e4m3(qx.codes).double()
    b = coat.decode_e4m3(qw.codes).double()
    s = float(qx.scales.float()) * float(qw.scales.float())
    ref = (a @ b) * s
    bound = (a.abs() @ b.abs()) * s * TAU + 1e-30
    r = _ratio(y, ref, bound)
    print(f"fp8_linear {M}x{K}x{N}: max err / (tau*sum|ab|) = {r:.3g}")
    assert r <= 1.0


def test_fp8_linear_matches_reference_loop(coat, port):
    """Against the C restatement of flow.cpp:21-33 (sequential fp32 loop)."""
    import torch
    M, K, N = 128, 512, 256
    qx, qw = _quant_pair(coat, M, K, N, seed=5)
    y = coat.fp8_linear(qx, qw).cpu().numpy()
    xd = coat.dequantize(qx).cpu().numpy()
    wd = coat.dequantize(qw).cpu().numpy()
    ref = port.matmul(xd, wd)
    bound = np.abs(xd).astype(np.float64) @ np.abs(wd).astype(np.float64)
    ratio = np.max(np.abs(y.astype(np.float64) - ref) / np.maximum(bound * TAU, 1e-300))
    print("vs reference loop:", ratio)
    assert ratio <= 1.0
    assert np.mean(y == ref) > 0.05   # many outputs bit-identical to the sequential loop


@pytest.mark.parametrize("M,K,N", [(16, 32, 16), (256, 512, 768), (600, 256, 512), (200, 272, 400),
                                   (8192, 5120, 13824)])   # 272: a partial 32-column bf16 output chunk
def test_linear_dgrad(coat, M, K, N):
    import torch
    qx, qw = _quant_pair(coat, M, K, N, seed=11)
    g = torch.Generator(device="cuda").manual_seed(13)
    dy = (torch.randn(M, N, device="cuda", generator=g) * 1e-3).to(torch.bfloat16)
    dx = coat.linear_dgrad(dy, qw)
    torch.cuda.synchronize()
    wu = coat.dequantize(qw).double()                          # W_used (K, N)
    ref = dy.double() @ wu.t()
    bound = (dy.double().abs() @ wu.abs().t()) * TAU
    err = (dx.double() - ref).abs()
    ok = err <= ref.abs() * 2.0 ** -8 + bound + 1e-30          # bf16 output rounding + accumulation
    assert bool(ok.all()), float((err - ref.abs() * 2.0 ** -8).max())


@pytest.mark.parametrize("M,K,N", [(16, 32, 16), (384, 256, 512), (608, 1280, 512), (208, 272, 400),
                                   (8192, 5120, 13824)])
def test_linear_wgrad(coat, M, K, N):
    import torch
    qx, qw = _quant_pair(coat, M, K, N, seed=17)
    g = torch.Generator(device="cuda").manual_seed(19)
    dy = (torch.randn(M, N, device="cuda", generator=g) * 1e-3).to(torch.bfloat16)
    dw = coat.linear_wgrad(qx, dy)
    torch.cuda.synchronize()
    xu = coat.dequantize(qx).double()                          # X_used (M, K)
    ref = xu.t() @ dy.double()
    tau = TAU * max(1.0, (M / 5120) ** 0.5)   # the reduction runs over M here
    bound = (xu.abs().t() @ dy.double().abs()) * tau + 1e-30
    r = _ratio(dw, ref, bound)
    print("wgrad ratio", r)
    assert r <= 1.0


def test_linear_errors(coat):
    import torch
    qx, qw = _quant_pair(coat, 128, 256, 256, seed=1)
    qbad = coat.quantize(torch.randn(128, 128, device="cuda"), coat.QuantGeometry.per_tensor())
    with pytest.raises(coat.ShapeMismatch):
        coat.fp8_linear(qx, qbad)
    qg = coat.quantize(torch.randn(128, 256, device="cuda"), coat.QuantGeometry.per_group(16))
    with pytest.raises(coat.InvalidSpec):
        coat.fp8_linear(qg, qw)


# ------------------------------------------------ quantizing GEMM epilogues ----
# SURVEY.md 8(f)#2 / PAPER.md:661-662: the per-group (1x16) quantizer of a GEMM
# output runs in the tcgen05 epilogue.  Parity: the codes and scales equal the
# oracle's quantize(y, 16) (quantize.cpp:89-111) applied to the kernel's own
# fp32 y, which the epilogue optionally writes beside them and which must be
# bit-identical to the plain forward GEMM's output.

def _np(t):
    return t.detach().cpu().numpy()


@pytest.mark.parametrize("M,K,N", [(16, 32, 128), (128, 256, 256), (200, 272, 400), (512, 1024, 768),
                                   (8192, 4096, 11008)])
def test_fp8_linear_q16_epilogue(coat, port, M, K, N):
    import torch
    qx, qw = _quant_pair(coat, M, K, N, seed=M + 3 * N)
    y_ref = coat.fp8_linear(qx, qw)
    q, y = coat.fp8_linear_q16(qx, qw, return_y=True)
    q_only = coat.fp8_linear_q16(qx, qw)
    torch.cuda.synchronize()
    assert torch.equal(y.view(torch.int32), y_ref.view(torch.int32)), "epilogue y differs from the forward GEMM"
    assert torch.equal(q.codes, q_only.codes) and torch.equal(q.scales, q_only.scales)
    rows = slice(None) if M * N <= (1 << 22) else slice(0, 256)   # the oracle on a row sample at full size
    yh = _np(y)[rows]
    codes, scales = port.quantize(yh, 16)
    assert np.array_equal(_np(q.codes)[rows], codes)
    assert np.array_equal(_np(q.scales.float()).reshape(M, N // 16)[rows].ravel(), scales)
    qd = coat.quantize(y, coat.QuantGeometry.per_group(16))   # the standalone device quantizer, every row
    assert torch.equal(q.codes, qd.codes) and torch.equal(q.scales, qd.scales)


# I % 128 == 0 takes the staged TMA-store epilogue (300 x 384: ragged rows), the others direct stores
@pytest.mark.parametrize("M,H,I", [(16, 32, 128), (128, 256, 256), (200, 272, 400), (300, 256, 384), (384, 512, 1040),
                                   (8192, 4096, 11008)])
def test_fp8_upgate_silu_epilogue(coat, port, M, H, I):
    """The fused gate/up GEMM + SiLU*mul quantizers == the two forward GEMMs
    followed by the SiLU*mul block (itself checked against the reference's
    DecoderLayer tape in test_gpu_producers.py), bit for bit; silu.in and
    mul.in.up also against the oracle's quantize on the GEMM outputs."""
    import torch
    qx, qwg = _quant_pair(coat, M, H, I, seed=7 * M + I)
    _, qwu = _quant_pair(coat, M, H, I, seed=7 * M + I + 1)
    gate = coat.fp8_linear(qx, qwg)
    up = coat.fp8_linear(qx, qwu)
    ref = coat.silu_mul_quantize(gate, up, return_prod=True)
    out = coat.fp8_upgate_silu(qx, qwg, qwu, return_fp32=True)
    fused = coat.fp8_upgate_silu(qx, qwg, qwu)
    torch.cuda.synchronize()
    g, u, p = out[4], out[5], out[6]
    assert torch.equal(g.view(torch.int32), gate.view(torch.int32))
    assert torch.equal(u.view(torch.int32), up.view(torch.int32))
    for a, b, c in zip(out[:4], ref[:4], fused):
        assert torch.equal(a.codes, b.codes) and torch.equal(a.scales, b.scales)
        assert torch.equal(c.codes, b.codes) and torch.equal(c.scales, b.scales)
    assert torch.equal(p.view(torch.int32), ref[4].view(torch.int32))
    rows = slice(None) if M * I <= (1 << 22) else slice(0, 128)
    for rec, src in ((out[0], gate), (out[2], up)):
        codes, scales = port.quantize(_np(src)[rows], 16)
        assert np.array_equal(_np(rec.codes)[rows], codes)
        assert np.array_equal(_np(rec.scales.float()).reshape(M, I // 16)[rows].ravel(), scales)


def test_quantizing_epilogue_nonfinite(coat):
    """A NaN code in x (E4M3 0x7F) makes y non-finite: quantize throws
    NonFiniteInput (quantize.cpp:91), so both epilogues raise it."""
    import torch
    qx, qw = _quant_pair(coat, 256, 256, 256, seed=3)
    qx.codes[17, 5] = 0x7F
    with pytest.raises(coat.NonFiniteInput):
        coat.fp8_linear_q16(qx, qw)
    with pytest.raises(coat.NonFiniteInput):
        coat.fp8_upgate_silu(qx, qw, qw)
    with pytest.raises(coat.GeometryMismatch):
        qa, qb = _quant_pair(coat, 128, 256, 264, seed=4)   # N % 16 != 0 is rejected
        coat.fp8_linear_q16(qa, qb)
