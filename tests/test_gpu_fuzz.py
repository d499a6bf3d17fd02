"""GPU: seeded fuzzing of the hot path against the oracle, bit for bit.

Random sizes (ragged, multi-round), random magnitude mixes per 1x128 group
(normal, log-uniform over many decades, tiny / huge, +-0 runs, constant groups,
outliers) and random optimizer states; every case is deterministic (seeded).
K1 (optimizer.cpp:101-114), the MGAQ quantizers (quantize.cpp:89-145) and the
DRE round trip (expand.cpp:100-141).  Found-bug regressions live in the
per-component test files; this sweeps the space around them.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CFG = {"beta1": 0.9, "beta2": 0.999, "lr": 1e-3, "weight_decay": 0.1, "eps": 1e-8}


def _dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _host(t):
    import torch
    return (t.float() if t.dtype == torch.bfloat16 else t).cpu().numpy()


def _mixed(r, n, scale=1.0):
    """n float32 values, a different distribution per 128-group."""
    out = np.empty(n, np.float32)
    for g0 in range(0, n, 128):
        k = min(128, n - g0)
        kind = r.integers(0, 8)
        if kind == 0:
            x = r.standard_normal(k)
        elif kind == 1:
            x = np.exp(r.uniform(-20, 5, k)) * r.choice([-1, 1], k)
        elif kind == 2:
            x = np.full(k, r.uniform(-2, 2))
        elif kind == 3:
            x = r.standard_normal(k) * 10.0 ** r.uniform(-30, -20)
        elif kind == 4:
            x = r.standard_normal(k) * 10.0 ** r.uniform(10, 25)
        elif kind == 5:
            x = r.standard_normal(k)
            x[r.random(k) < 0.5] = 0.0
            x[r.random(k) < 0.2] = -0.0
        elif kind == 6:
            x = r.standard_normal(k)
            x[r.integers(0, k)] *= 1e4
        else:
            x = np.exp(r.uniform(-3, 3, k))
        out[g0:g0 + k] = (np.asarray(x) * scale).astype(np.float32)
    return out


@pytest.mark.parametrize("case", range(40))
def test_fuzz_k1_steps(coat, port, checker, case):
    r = np.random.default_rng(1000 + case)
    n = int(r.choice([128 * r.integers(1, 40), 1792 * r.integers(1, 200) + r.integers(0, 1792),
                      int(r.integers(1000, 400_000))]))
    w = _mixed(r, n, 0.02)
    m, v = checker.make_slot(n)
    slot = coat.make_slot([n])
    wg = _dev(w)
    cfg = dict(CFG, weight_decay=float(r.choice([0.0, 0.1])), lr=float(r.choice([1e-3, 1e-4])))
    c = coat.AdamWConfig(**cfg)
    for t in range(int(r.integers(1, 4))):
        g = _mixed(r, n, float(r.choice([1e-3, 1.0, 1e-6])))
        if t == 0:   # the first step always compares fully: keep g*g finite
            g = np.clip(np.nan_to_num(g, posinf=0.0, neginf=0.0), -1e15, 1e15).astype(np.float32)
        st = checker.step(w, g, m, v, t, cfg)
        assert t > 0 or st == 0, (case, st)
        if st != 0:   # the reference throws (e.g. g*g overflow -> NonFiniteInput): so must the GPU
            with pytest.raises(Exception):
                coat.step(wg, _dev(g), slot, c)
            return
        coat.step(wg, _dev(g), slot, c)
        assert np.array_equal(_host(wg).view(np.uint32), w.view(np.uint32)), (case, t)
        for st_, ref in ((slot.m, m), (slot.v, v)):
            assert np.array_equal(_host(st_.quantized.codes), ref["codes"]), (case, t)
            assert np.array_equal(_host(st_.quantized.scales), ref["scales"]), (case, t)
            assert np.array_equal(_host(st_.k).view(np.uint32), ref["k"].view(np.uint32)), (case, t)
            assert np.array_equal(_host(st_.c).view(np.uint32), ref["c"].view(np.uint32)), (case, t)


@pytest.mark.parametrize("case", range(40))
def test_fuzz_mgaq(coat, port, checker, case):
    import torch
    r = np.random.default_rng(2000 + case)
    G = int(r.choice([0, 16, 32, 64, 128]))
    cols = int(r.choice([16, 48, 128, 384, 4096, 11008])) if G in (0, 16) else int(G * r.integers(1, 40))
    rows = int(r.integers(1, 300))
    x = _mixed(r, rows * cols).reshape(rows, cols)
    bf16 = bool(r.integers(0, 2))
    if bf16:
        xt = torch.from_numpy(x).to(torch.bfloat16)
        x = xt.float().numpy()
    else:
        xt = torch.from_numpy(x)
    if not np.isfinite(x).all():
        return
    geo = coat.QuantGeometry.per_group(G) if G else coat.QuantGeometry.per_tensor()
    q = coat.quantize(xt.cuda(), geo)
    codes, scales = checker.quantize(x, G)
    assert np.array_equal(_host(q.codes), codes), case
    assert np.array_equal(_host(q.scales).ravel(), np.asarray(scales).ravel()), case


@pytest.mark.parametrize("case", range(20))
def test_fuzz_dre_round_trip(coat, port, checker, case):
    r = np.random.default_rng(3000 + case)
    n = 128 * int(r.integers(1, 3000))
    x = _mixed(r, n, float(r.choice([1e-6, 1.0, 1e-30])))
    st = coat.expand_quantize(_dev(x))
    codes, s, k, c = checker.expand_quantize(x)
    assert np.array_equal(_host(st.quantized.codes), codes), case
    assert np.array_equal(_host(st.quantized.scales), s), case
    assert np.array_equal(_host(st.k).view(np.uint32), k.view(np.uint32)), case
    assert np.array_equal(_host(st.c).view(np.uint32), c.view(np.uint32)), case
    back = _host(coat.dequantize_contract(st))
    assert np.array_equal(back.view(np.uint32), checker.dequantize_contract(codes, s, k, c).view(np.uint32)), case


def _moment_state(port, r, n, positive):
    x = _mixed(r, n, float(r.choice([1e-3, 1e-8, 1e-20, 1.0])))
    if positive:
        x = np.abs(x)
    x = np.nan_to_num(x, posinf=0.0, neginf=0.0).astype(np.float32)
    codes, s, k, c = port.expand_quantize(x)
    return {"codes": codes, "scales": s, "k": k, "c": c}


@pytest.mark.parametrize("case", range(40))
def test_fuzz_k1_warm_states(coat, port, checker, case):
    """K1 from random warm states (m, v built by the oracle's expand_quantize of
    mixed distributions: k spread over [1, 20], tiny and huge scales), random
    step counters and AdamW settings."""
    r = np.random.default_rng(4000 + case)
    n = 128 * int(r.integers(1, 2500))
    w = _mixed(r, n, float(r.choice([0.02, 1.0, 1e-6])))
    w = np.clip(np.nan_to_num(w, posinf=0.0, neginf=0.0), -1e30, 1e30).astype(np.float32)
    m = _moment_state(checker, r, n, False)
    v = _moment_state(checker, r, n, True)
    t0 = int(r.integers(0, 10000))
    cfg = {"beta1": float(r.choice([0.9, 0.8, 0.95])), "beta2": float(r.choice([0.999, 0.99, 0.95])),
           "lr": float(r.choice([1e-3, 3e-4, 1e-2])), "weight_decay": float(r.choice([0.0, 0.1, 0.01])),
           "eps": float(r.choice([1e-8, 1e-6, 1e-12]))}
    slot = coat.make_slot([n])
    slot.load_state(m, v, t0)
    wg = _dev(w)
    g = _mixed(r, n, float(r.choice([1e-3, 1e-6, 1e-12])))
    g = np.clip(np.nan_to_num(g, posinf=0.0, neginf=0.0), -1e15, 1e15).astype(np.float32)
    st = checker.step(w, g, m, v, t0, cfg)
    if st != 0:
        with pytest.raises(Exception):
            coat.step(wg, _dev(g), slot, coat.AdamWConfig(**cfg))
        return
    coat.step(wg, _dev(g), slot, coat.AdamWConfig(**cfg))
    assert np.array_equal(_host(wg).view(np.uint32), w.view(np.uint32)), case
    for st_, ref in ((slot.m, m), (slot.v, v)):
        assert np.array_equal(_host(st_.quantized.codes), ref["codes"]), case
        assert np.array_equal(_host(st_.quantized.scales), ref["scales"]), case
        assert np.array_equal(_host(st_.k).view(np.uint32), ref["k"].view(np.uint32)), case
        assert np.array_equal(_host(st_.c).view(np.uint32), ref["c"].view(np.uint32)), case


@pytest.mark.parametrize("case", range(16))
def test_fuzz_rmsnorm_block(coat, port, case):
    import torch
    r = np.random.default_rng(5000 + case)
    rows, h = int(r.integers(1, 200)), int(16 * r.integers(1, 300))
    x = _mixed(r, rows * h, float(r.choice([1.0, 1e-3, 30.0]))).reshape(rows, h)
    x = np.clip(np.nan_to_num(x, posinf=0.0, neginf=0.0), -1e18, 1e18).astype(np.float32)
    xt = torch.from_numpy(x).to(torch.bfloat16)
    x = xt.float().numpy()
    w = (1.0 + 0.2 * r.standard_normal(h)).astype(np.float32)
    qx, qy, rms, y = coat.rmsnorm_quantize(xt.cuda(), torch.from_numpy(w), eps=1e-6, return_y=True)
    xc, xs = port.quantize(x, 16)
    assert np.array_equal(_host(qx.codes), xc) and np.array_equal(_host(qx.scales).ravel(), xs.ravel()), case
    y_ref = port.rmsnorm(port.dequantize(xc, xs, 16), w, 1e-6)
    assert np.array_equal(_host(y).view(np.uint32), y_ref.view(np.uint32)), case


@pytest.mark.parametrize("case", range(16))
def test_fuzz_silu_mul_block(coat, port, case):
    """Random (rows, cols) -- chunk counts that leave the last warp partly
    filled -- and gate magnitudes that reach silu's large-|x| branch."""
    import torch
    r = np.random.default_rng(6000 + case)
    rows, cols = int(r.integers(1, 200)), int(16 * r.integers(1, 300))
    g = _mixed(r, rows * cols, float(r.choice([1.0, 30.0, 1e-3]))).reshape(rows, cols)
    u = _mixed(r, rows * cols, float(r.choice([1.0, 1e-2]))).reshape(rows, cols)
    g = np.clip(np.nan_to_num(g, posinf=0.0, neginf=0.0), -1e4, 1e4).astype(np.float32)
    u = np.clip(np.nan_to_num(u, posinf=0.0, neginf=0.0), -1e4, 1e4).astype(np.float32)
    gt, ut = torch.from_numpy(g).to(torch.bfloat16), torch.from_numpy(u).to(torch.bfloat16)
    gn, un = gt.float().numpy(), ut.float().numpy()
    qg, qs, qu, qp, prod = coat.silu_mul_quantize(gt.cuda(), ut.cuda(), return_prod=True)
    gc, gs = port.quantize(gn, 16)
    uc, us = port.quantize(un, 16)
    assert np.array_equal(_host(qg.codes), gc) and np.array_equal(_host(qg.scales).ravel(), gs.ravel()), case
    assert np.array_equal(_host(qu.codes), uc) and np.array_equal(_host(qu.scales).ravel(), us.ravel()), case
    s_dq = port.dequantize(_host(qs.codes), _host(qs.scales), 16)
    p_ref = (s_dq * port.dequantize(uc, us, 16)).astype(np.float32)
    assert np.array_equal(_host(prod).view(np.uint32), p_ref.view(np.uint32)), case
    pc, ps = port.quantize(p_ref, 0)
    assert np.array_equal(_host(qp.codes), pc) and np.array_equal(_host(qp.scales).ravel(), np.asarray(ps).ravel()), case
    sc, _ = port.quantize(port.silu(port.dequantize(gc, gs, 16)), 16)
    assert np.count_nonzero(_host(qs.codes) != sc) <= max(2, sc.size // 1000), case
