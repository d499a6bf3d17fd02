"""GPU: the K1 pack warp's low-latency pack_prepare (dre_fast.cuh
pack_prepare_lowlat: certified FP64 approximations + exact fallback) equals
the exact pack_prepare_fast bit for bit -- k, c, the BF16 group scale, RN(1/c),
RN(1/s), the pack mode and the NonFiniteInput bit -- on random and adversarial
group extrema.  pack_prepare_fast itself is pinned to the reference through the
K1 parity tests (measure_group + optimal_k + group scale, expand.cpp:50-83,
quantize.cpp:10-17).
"""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

LOG_TARGET = math.log(229376.0)   # expand.cpp:52


def _run(lo_bits, hi_bits):
    import torch
    from paper_2410_19313_b200 import _lib
    lo = torch.from_numpy(np.ascontiguousarray(lo_bits, dtype=np.uint32).view(np.int32)).cuda()
    hi = torch.from_numpy(np.ascontiguousarray(hi_bits, dtype=np.uint32).view(np.int32)).cuda()
    n = lo.numel()
    out = torch.empty(n * 14, dtype=torch.float32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    assert _lib.lib.coat_test_pack_prepare(lo.data_ptr(), hi.data_ptr(), n, LOG_TARGET, out.data_ptr(), st) == 0
    torch.cuda.synchronize()
    o = out.cpu().numpy().view(np.uint32).reshape(n, 2, 7)
    return o[:, 0], o[:, 1]


def _check(lo_bits, hi_bits):
    fast, exact = _run(lo_bits, hi_bits)
    bad = np.nonzero((fast != exact).any(axis=1))[0]
    if bad.size:
        i = bad[0]
        f = lambda b: np.uint32(b).view(np.float32)  # noqa: E731
        raise AssertionError(
            f"{bad.size} of {len(lo_bits)} differ; first lo={f(lo_bits[i])!r} hi={f(hi_bits[i])!r}\n"
            f"lowlat={fast[i].view(np.float32)}\nexact ={exact[i].view(np.float32)}")
    return exact


def _bits(x):
    return np.asarray(x, dtype=np.float32).view(np.uint32)


def test_random_moment_like_extrema():
    rng = np.random.default_rng(7)
    n = 1 << 22
    hi = np.exp2(rng.uniform(-60.0, 10.0, n)).astype(np.float32)
    ratio = np.exp2(rng.uniform(0.0, 40.0, n))
    lo = np.maximum((hi / ratio).astype(np.float32), np.float32(1e-45))
    lo = np.minimum(lo, hi)
    ex = _check(_bits(lo), _bits(hi))
    modes = ex[:, 5].view(np.float32)
    assert (modes == 0).any() and (modes == 1).any()   # both scale paths exercised


def test_random_full_float_range():
    rng = np.random.default_rng(11)
    n = 1 << 22
    a = rng.integers(1, 0x7F800000, n, dtype=np.uint32)
    b = rng.integers(1, 0x7F800000, n, dtype=np.uint32)
    _check(np.minimum(a, b), np.maximum(a, b))


def test_clamp_and_rounding_boundaries():
    rng = np.random.default_rng(3)
    n = 1 << 20
    hi = np.exp2(rng.uniform(-40.0, 5.0, n)).astype(np.float32)
    l2t = LOG_TARGET / math.log(2.0)
    cases = []
    # k = log_target / log(range) near 1 (range ~ 229376) and near kMax = 20 (range ~ 1.853)
    for center in (l2t, l2t / 20.0):
        r = np.exp2(center * (1.0 + rng.uniform(-1e-6, 1e-6, n)))
        cases.append((hi, (hi / r).astype(np.float32)))
    # k whose float rounding is near a midpoint: L2 = l2t / k_mid for k_mid = midpoints of floats in (1, 20)
    kf = np.exp2(rng.uniform(0.0, math.log2(20.0), n)).astype(np.float32)
    kmid = kf.astype(np.float64) * (1.0 + 2.0 ** -24)
    r = np.exp2(l2t / kmid)
    cases.append((hi, (hi / r).astype(np.float32)))
    for h, lo in cases:
        lo = np.minimum(np.maximum(lo, np.float32(1e-45)), h)
        _check(_bits(lo), _bits(h))


def test_special_extrema():
    f32 = np.float32
    vals = [(1.0, 1.0), (1.0, np.nextafter(f32(1.0), f32(2.0))), (0.0, 0.0), (1e-45, 1e-45), (1e-45, 3.4e38),
            (1e-30, 1e-30), (1e-38, 1e-20), (1e-40, 1e-39), (2.0 ** -100, 2.0 ** -100), (2.0 ** -101, 2.0 ** -99),
            (1e30, 3.4e38), (2.0 ** 100, 2.0 ** 100), (2.0 ** 101, 2.0 ** 101), (1.0, 448.0), (1.0, 229376.0),
            (3.0, 3.0 * 229376.0), (1e-3, 1e-3 * 1.853), (5e-8, 7e-3), (1e-12, 2.5e-6)]
    lo = [_bits(f32(a)) for a, _ in vals]
    hi = [_bits(f32(b)) for _, b in vals]
    lo += [np.uint32(0x3F800000), np.uint32(0x00000001), np.uint32(0x3F800000)]
    hi += [np.uint32(0x7F800000), np.uint32(0x7FC00000), np.uint32(0x7F7FFFFF)]   # Inf, NaN, FLT_MAX
    _check(np.array(lo, dtype=np.uint32), np.array(hi, dtype=np.uint32))


def test_mufu_error_bounds():
    """The error model behind the DRE pack's flat 2^-15 certification interval
    (dre.cuh kRelMufu; k1_ws.cu pack4_sfu), exhaustively on this hardware:
    lg2.approx.ftz(r) is within 2^-22 * (1 + |log2 r|) of log2(r) for every
    float r in [2^-10, 2^10] (r = |x| * RN(1/c): |x|/c in [2^-9, 2^9] by
    measure_group), and ex2.approx.ftz(u) within 2^-22 (relative) of 2^u for
    every float |u| < 9.5 (|u| = |k log2(|x|/c)| <= 8.95).  Then q = RN(RN(ex2(
    RN(k * lg2(RN(|x| RN(1/c)))))) RN(1/s)) has relative error <= ln2 * (k *
    2^-22 + 8.95 * 2^-22 + 8.95 * 2^-24) + k * 2^-23 + 2^-22 + 2^-23 < 2^-16.9
    for k <= 20: the interval keeps a 3.7x margin."""
    import torch
    from paper_2410_19313_b200 import _lib
    out = torch.zeros(2, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    assert _lib.lib.coat_test_mufu_bounds(2.0 ** -10, 2.0 ** 10, 9.5, out.data_ptr(), st) == 0
    torch.cuda.synchronize()
    e_lg, e_ex = out.cpu().numpy().view(np.float64)
    print(f"lg2.approx max err / (1 + |log2 r|) 2^{math.log2(e_lg):.2f}, ex2.approx max rel err "
          f"2^{math.log2(e_ex):.2f}")
    assert e_lg <= 2.0 ** -22 and e_ex <= 2.0 ** -22

