"""GPU parity: Dynamic Range Expansion quantize / contract vs the CPU oracle.

Reference: expand.cpp:18-141 (measure_group, optimal_k, expand, contract,
expand_quantize, dequantize_contract).  Bit-exact: codes, BF16 scales, k, c and
the contracted fp32 values.
"""
import numpy as np
import pytest

from conftest import rng

pytestmark = pytest.mark.gpu


def dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    import torch
    return (t.float() if t.dtype == torch.bfloat16 else t).cpu().numpy()


def m_like(port, groups, seed=21, frac=0.01):
    return port.generate(0, (groups * 128,), frac, 100.0, seed) * np.float32(1e-4)


def v_like(groups, seed=22):
    r = rng(seed)
    out = []
    for q in r.uniform(2.5, 11.0, groups):
        out.append(np.exp(r.uniform(-0.5 * np.log(q), 0.5 * np.log(q), 128)) * 1e-8)
    return np.concatenate(out).astype(np.float32)


def special_groups():
    g = []
    g.append(np.zeros(128, np.float32))                        # all zero -> degenerate
    g.append(np.full(128, 0.25, np.float32))                   # constant -> degenerate
    x = np.full(128, 2.0 ** -9, np.float32); x[0] = 448; g.append(x)  # exactly the E4M3 range
    x = np.zeros(128, np.float32); x[3] = -1e-3; g.append(x)   # single nonzero
    x = np.linspace(1, 1.01, 128).astype(np.float32); g.append(x)   # k clamps to 20
    x = np.geomspace(1e-30, 1e10, 128).astype(np.float32); g.append(x)  # k clamps to 1
    x = np.full(128, -3.0, np.float32); x[::2] = 3.0; g.append(x)
    x = rng(5).standard_normal(128).astype(np.float32); x[::3] = 0; g.append(x)
    tiny = np.geomspace(1e-38, 1e-36, 128).astype(np.float32); g.append(tiny)   # tiny scales
    big = np.geomspace(1e30, 3e38, 128).astype(np.float32); g.append(big)
    g.append(np.full(128, -0.0, np.float32))                   # all -0 (expand_one(-0) = +0)
    x = np.geomspace(1e-45, 3e-44, 128).astype(np.float32); g.append(x)   # subnormal c with k > 1
    x = rng(6).standard_normal(128).astype(np.float32); x[1::4] = -0.0; g.append(x)   # -0 among values
    return np.concatenate(g)


def _check_state(coat, port, x):
    st = coat.expand_quantize(dev(x))
    codes, s, k, c = port.expand_quantize(x)
    got_codes = host(st.quantized.codes)
    bad = np.nonzero(got_codes != codes)[0]
    assert bad.size == 0, (bad[:10], got_codes[bad[:10]], codes[bad[:10]], x[bad[:10]])
    assert np.array_equal(host(st.quantized.scales), s)
    assert np.array_equal(host(st.k).view(np.uint32), k.view(np.uint32))
    assert np.array_equal(host(st.c).view(np.uint32), c.view(np.uint32))
    back = host(coat.dequantize_contract(st))
    exp = port.dequantize_contract(codes, s, k, c)
    diff = np.nonzero(back.view(np.uint32) != exp.view(np.uint32))[0]
    assert diff.size == 0, (diff[:10], back[diff[:10]], exp[diff[:10]])


def test_expand_quantize_m_like(coat, port, checker):
    _check_state(coat, checker, m_like(port, 4096))


def test_expand_quantize_v_like(coat, port, checker):
    _check_state(coat, checker, v_like(4096))


def test_expand_quantize_special_groups(coat, port, checker):
    _check_state(coat, checker, special_groups())


def test_expand_quantize_uniform_log(coat, port, checker):
    for rr, seed in ((1e2, 5), (1e4, 6), (1e6, 7), (2.0, 8)):
        _check_state(coat, checker, port.generate(2, (128 * 512,), 0.0, rr, seed))


def test_expand_quantize_large_random(coat, port, checker):
    """Many groups with k spread across [1, 20]: exactness at scale."""
    r = rng(1234)
    groups = 1 << 14
    ranges = np.exp(r.uniform(np.log(1.05), np.log(1e7), groups))
    x = np.concatenate([np.exp(r.uniform(-0.5 * np.log(q), 0.5 * np.log(q), 128))
                        * r.choice([-1, 1], 128) * 10 ** r.uniform(-9, 2) for q in ranges])
    _check_state(coat, checker, x.astype(np.float32))


def test_expand_quantize_cfg1_size(coat, port):
    """cfg1's 16 Mi-element moment tensors (131,072 groups), m-like and v-like."""
    groups = 1 << 17
    _check_state(coat, port, m_like(port, groups, seed=41))
    _check_state(coat, port, v_like(groups, seed=42))


def test_fallback_rate_is_small(coat, port):
    import torch
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    coat.set_fallback_counter(cnt)
    try:
        x = np.concatenate([m_like(port, 2048), v_like(2048)])
        coat.expand_quantize(dev(x))
        torch.cuda.synchronize()
        rate = int(cnt.item()) / x.size
    finally:
        coat.set_fallback_counter(None)
    assert rate < 5e-3, rate


def test_dre_errors(coat):
    with pytest.raises(coat.GeometryMismatch):
        coat.expand_quantize(dev(np.ones(130, np.float32)))
    with pytest.raises(coat.InvalidSpec):
        coat.expand_quantize(dev(np.ones(128, np.float32)), group_size=64)
    x = np.ones(256, np.float32)
    x[200] = np.inf
    with pytest.raises(coat.NonFiniteInput):
        coat.expand_quantize(dev(x))
