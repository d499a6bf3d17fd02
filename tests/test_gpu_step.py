"""GPU parity: the fused FP8-DRE AdamW step (K1) vs coatsim::step.

Reference: optimizer.cpp:90-114 with the {E4M3, expand, 128} policy for both
moments.  Bit-exact on the updated fp32 weights, codes, BF16 scales, k and c,
over multi-step trajectories, ragged sizes and the error semantics.
"""
import numpy as np
import pytest

from conftest import rng

pytestmark = pytest.mark.gpu

CFG = {"beta1": 0.9, "beta2": 0.999, "lr": 1e-3, "weight_decay": 0.1, "eps": 1e-8}


def dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    import torch
    return (t.float() if t.dtype == torch.bfloat16 else t).cpu().numpy()


def gpu_state(slot):
    out = []
    for st in (slot.m, slot.v):
        out.append({"codes": host(st.quantized.codes), "scales": host(st.quantized.scales),
                    "k": host(st.k), "c": host(st.c)})
    return out


def assert_state_equal(got, exp, what=""):
    for key in ("codes", "scales", "k", "c"):
        a, b = got[key], exp[key]
        bad = np.nonzero(a.view(np.uint8 if key == "codes" else np.uint32)
                         != b.view(np.uint8 if key == "codes" else np.uint32))[0]
        assert bad.size == 0, (what, key, bad[:8], a[bad[:8]], b[bad[:8]])


def run_both(coat, port, n, steps, cfg=CFG, seed=1, warm=None, grad_scale=1e-3, t_start=9):
    w0 = port.generate(0, (n,), 0.0, 100.0, seed) * np.float32(0.02)
    w_ref = w0.copy()
    m, v = port.make_slot(n)
    slot = coat.make_slot([n])
    if warm is not None:
        m, v = warm
        slot.load_state(m, v, t_start)
        m = {k: a.copy() for k, a in m.items()}
        v = {k: a.copy() for k, a in v.items()}
    t0 = slot.step
    w = dev(w0)
    c = coat.AdamWConfig(**cfg)
    for t in range(steps):
        g = port.generate(0, (n,), 0.01, 100.0, 100 + t) * np.float32(grad_scale)
        assert port.step(w_ref, g, m, v, t0 + t, cfg) == 0
        coat.step(w, dev(g), slot, c)
        gm, gv = gpu_state(slot)
        wd = host(w)
        bad = np.nonzero(wd.view(np.uint32) != w_ref.view(np.uint32))[0]
        assert bad.size == 0, (t, bad[:8], wd[bad[:8]], w_ref[bad[:8]])
        assert_state_equal(gm, m, f"m step {t}")
        assert_state_equal(gv, v, f"v step {t}")
    assert slot.step == t0 + steps


@pytest.mark.parametrize("n", [128, 512, 4096, 5000, 1000 * 128 + 3, 1 << 16])
def test_step_trajectory_bit_exact(coat, port, checker, n):
    run_both(coat, checker, n, 5)


@pytest.mark.parametrize("t_start", [9, 160, 20000])
def test_step_from_warmed_state(coat, port, checker, t_start):
    """Fixture (B) of SURVEY.md 8(d): m with k ~ 1-3, v with k ~ 5-15, t = 10;
    also late in a run: t = 161 (bc1 one ulp below 1) and t = 20001 (bc1 =
    bc2 = 1 exactly in fp32: the Markstein divisions by 1)."""
    groups = 2048
    n = groups * 128
    m0 = port.generate(0, (n,), 0.01, 100.0, 21) * np.float32(1e-4)
    r = rng(22)
    v0 = np.concatenate([np.exp(r.uniform(-0.5 * np.log(q), 0.5 * np.log(q), 128)) * 1e-8
                         for q in r.uniform(2.5, 11.0, groups)]).astype(np.float32)
    mc, ms, mk, mcc = checker.expand_quantize(m0)
    vc, vs, vk, vcc = checker.expand_quantize(v0)
    warm = ({"codes": mc, "scales": ms, "k": mk, "c": mcc}, {"codes": vc, "scales": vs, "k": vk, "c": vcc})
    run_both(coat, checker, n, 3, warm=warm, t_start=t_start)


def test_step_sparse_zero_and_extreme_groups(coat, port, checker):
    """Groups the fast paths must hand off exactly: whole zero groups (v' == 0,
    all-zero state), scattered zero gradients (zero-aware extrema), tiny and
    huge gradient groups (IEEE AdamW path, literal contract/pack), through
    several steps so k == 1 and k > 1 states both reach the contract."""
    n = 96 * 2048 + 640
    w0 = port.generate(0, (n,), 0.0, 100.0, 5) * np.float32(0.02)
    w_ref = w0.copy()
    m, v = checker.make_slot(n)
    slot = coat.make_slot([n])
    w = dev(w0)
    c = coat.AdamWConfig(**CFG)
    r = rng(77)
    for t in range(6):
        g = port.generate(0, (n,), 0.01, 100.0, 300 + t) * np.float32(1e-3)
        gv = g.reshape(-1, 128)
        gv[r.random(gv.shape[0]) < 0.15] = 0.0                    # untouched rows
        gv[r.random(gv.shape) < 0.05] = 0.0                       # scattered zeros
        gv[3::41] *= np.float32(1e-30)                            # tiny groups
        gv[5::53] *= np.float32(1e16)                             # huge groups
        gv[7::59, :64] = 0.0
        assert checker.step(w_ref, g, m, v, t, CFG) == 0
        coat.step(w, dev(g), slot, c)
        gm, gvs = gpu_state(slot)
        wd = host(w)
        bad = np.nonzero(wd.view(np.uint32) != w_ref.view(np.uint32))[0]
        assert bad.size == 0, (t, bad[:8], wd[bad[:8]], w_ref[bad[:8]])
        assert_state_equal(gm, m, f"m step {t}")
        assert_state_equal(gvs, v, f"v step {t}")


def test_step_without_weight_decay_and_large_grads(coat, port, checker):
    run_both(coat, checker, 1 << 14, 3, cfg=dict(CFG, weight_decay=0.0), grad_scale=1.0)


def test_step_kat_first_step(coat):
    """t = 1, g = 1, zero state -> w - lr/(1+eps) per element (wd = 0)."""
    import torch
    n = 1024
    slot = coat.make_slot([n])
    w = torch.zeros(n, device="cuda")
    coat.step(w, torch.ones(n, device="cuda"), slot, coat.AdamWConfig(lr=1e-3))
    expect = np.float32(0) - np.float32(1e-3) * (np.float32(1) / (np.float32(1) + np.float32(1e-8)))
    assert np.all(host(w) == expect)


def test_nonfinite_grad_leaves_everything_untouched(coat):
    import torch
    n = 4096
    slot = coat.make_slot([n])
    w = torch.randn(n, device="cuda")
    c = coat.AdamWConfig(weight_decay=0.1)
    coat.step(w, torch.randn(n, device="cuda") * 1e-3, slot, c)
    w_before = w.clone()
    m_before = slot.m.quantized.codes.clone()
    g = torch.randn(n, device="cuda")
    g[1234] = float("nan")
    with pytest.raises(coat.NonFiniteGradient):
        coat.step(w, g, slot, c)
    assert torch.equal(w, w_before) and torch.equal(slot.m.quantized.codes, m_before)
    assert slot.step == 1


def test_pack_failure_commits_like_reference(coat, port, checker):
    """g*g overflow -> v = inf -> pack_moment(v) throws: params and m committed,
    v and the step counter not (optimizer.cpp:101-114)."""
    import torch
    n = 512
    slot = coat.make_slot([n])
    w = torch.ones(n, device="cuda")
    g = torch.zeros(n, device="cuda")
    g[3] = 1e20
    v_before = slot.v.quantized.codes.clone()
    with pytest.raises(coat.NonFiniteInput):
        coat.step(w, g, slot, coat.AdamWConfig(weight_decay=0.1))
    # reference
    wr = np.ones(n, np.float32)
    m, v = checker.make_slot(n)
    m0 = {k: a.copy() for k, a in m.items()}
    assert checker.step(wr, host(g), m, v, 0, dict(CFG)) == 3
    assert np.array_equal(host(w), wr)
    assert torch.equal(slot.v.quantized.codes, v_before)
    assert np.array_equal(host(slot.m.quantized.codes), m["codes"])
    assert slot.step == 0


def test_shape_and_policy_errors(coat):
    import torch
    slot = coat.make_slot([256])
    with pytest.raises(coat.ShapeMismatch):
        coat.step(torch.zeros(255, device="cuda"), torch.zeros(255, device="cuda"), slot, coat.AdamWConfig())
    with pytest.raises(coat.ShapeMismatch):
        coat.step(torch.zeros(256, device="cuda"), torch.zeros(128, device="cuda"), slot, coat.AdamWConfig())
    with pytest.raises(coat.InvalidSpec):
        coat.make_slot([256], coat.SlotPolicy(coat.MomentPolicy(coat.StateFormat.DE8)))


def test_step_16m_against_multithreaded_reference(coat, ref):
    """Config 1 size (2^24 params), two steps from zero state + warmed state,
    against the unmodified reference run on all host cores."""
    import os
    n = 1 << 24
    th = os.cpu_count() or 8
    w0 = ref.generate(0, (n,), 0.0, 100.0, 1) * np.float32(0.02)
    w_ref = w0.copy()
    m, v = ref.make_slot(n)
    slot = coat.make_slot([n])
    w = dev(w0)
    c = coat.AdamWConfig(**CFG)
    for t in range(2):
        g = ref.generate(0, (n,), 0.01, 100.0, 100 + t) * np.float32(1e-3)
        assert ref.step(w_ref, g, m, v, t, CFG, threads=th) == 0
        coat.step(w, dev(g), slot, c)
    gm, gv = gpu_state(slot)
    assert np.array_equal(host(w).view(np.uint32), w_ref.view(np.uint32))
    assert_state_equal(gm, m, "m")
    assert_state_equal(gv, v, "v")


def test_step_in_place_state_matches_ping_pong(coat, port):
    """coat_adamw_dre_step with w_out == w_in and m_out == m_in, v_out == v_in
    (aliasing allowed) gives the same weights and state as the
    ping-pong buffers the Python mirror uses.  The round pipeline only prefetches
    rounds ahead of the ones it writes back, so in-place is exact; 3.2M params
    = many rounds per CTA, with a ragged tail."""
    import ctypes as C
    import torch
    from paper_2410_19313_b200 import _lib
    L = _lib.lib
    n = 25 * 1792 * 72 + 128 * 5 + 77
    ng = -(-n // 128)
    r = rng(31)
    w0 = (r.standard_normal(n) * 0.02).astype(np.float32)

    def moment():
        return {"codes": torch.zeros(n, dtype=torch.uint8, device="cuda"),
                "scales": torch.full((ng,), 0x3F80, dtype=torch.int16, device="cuda"),
                "k": torch.ones(ng, device="cuda"), "c": torch.ones(ng, device="cuda")}

    def cs(mm):
        return _lib.MomentState(mm["codes"].data_ptr(), mm["scales"].data_ptr(), mm["k"].data_ptr(),
                                mm["c"].data_ptr())

    cfg = _lib.AdamWConfigC(**CFG)
    flags = torch.zeros(1, dtype=torch.int32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    # ping-pong
    wp = [dev(w0), torch.empty(n, device="cuda")]
    mp, vp = [moment(), moment()], [moment(), moment()]
    # in place
    wi, mi, vi = dev(w0), moment(), moment()
    for t in range(1, 5):
        g = dev((r.standard_normal(n) * 1e-3).astype(np.float32))
        a, b = (t - 1) % 2, t % 2
        assert L.coat_adamw_dre_step(wp[a].data_ptr(), wp[b].data_ptr(), g.data_ptr(), n, 128, cs(mp[a]),
                                     cs(vp[a]), cs(mp[b]), cs(vp[b]), C.byref(cfg), t, flags.data_ptr(), st) == 0
        assert L.coat_adamw_dre_step(wi.data_ptr(), wi.data_ptr(), g.data_ptr(), n, 128, cs(mi), cs(vi), cs(mi),
                                     cs(vi), C.byref(cfg), t, flags.data_ptr(), st) == 0
        torch.cuda.synchronize()
        assert int(flags.item()) == 0
        assert torch.equal(wi, wp[b]), t
        for x, y in ((mi, mp[b]), (vi, vp[b])):
            for key in ("codes", "scales", "k", "c"):
                assert torch.equal(x[key], y[key]), (t, key)


@pytest.mark.parametrize("moment,group,k,code", [("m", 3, 1.0, 0x7F), ("m", 5, 2.5, 0xFF),
                                                  ("v", 7, 3.0, 0x7F), ("v", 9, 1.0, 0xFF)])
def test_nan_code_in_state_is_a_contract_error(coat, port, checker, moment, group, k, code):
    """A NaN E4M3 code in the stored state (0x7F / 0xFF) makes unpack (decode,
    fp8.cpp:145-152) throw NonFiniteInput before anything is mutated -- for a
    k == 1 group (exact contract) and a k != 1 group (table contract, where the
    product itself would be finite), in m and in v; the reference agrees."""
    import torch
    n = 128 * 64
    r = rng(51)
    w0 = (r.standard_normal(n) * 0.02).astype(np.float32)
    g0 = (r.standard_normal(n) * 1e-3).astype(np.float32)
    m, v = checker.make_slot(n)
    wr = w0.copy()
    assert checker.step(wr, g0, m, v, 0, CFG) == 0
    st = {"m": m, "v": v}[moment]
    st["codes"][group * 128 + 17] = code
    st["k"][group] = np.float32(k)
    slot = coat.make_slot([n])
    slot.load_state(m, v, 1)
    w = dev(wr)
    g = dev((r.standard_normal(n) * 1e-3).astype(np.float32))
    before = [t.clone() for t in (w, slot.m.quantized.codes, slot.v.quantized.codes, slot.m.k, slot.v.k)]
    with pytest.raises(coat.NonFiniteInput):
        coat.step(w, g, slot, coat.AdamWConfig(**CFG))
    after = (w, slot.m.quantized.codes, slot.v.quantized.codes, slot.m.k, slot.v.k)
    assert all(torch.equal(a, b) for a, b in zip(after, before))
    assert slot.step == 1
    # the reference throws NonFiniteInput as well and leaves w untouched
    w_ref = wr.copy()
    assert checker.step(w_ref, host(g), m, v, 1, CFG) == 3
    assert np.array_equal(w_ref, wr)


def test_step_signed_zero_weights_and_grads(coat, port, checker):
    """w and g containing +0 and -0 (and groups of them) step exactly like
    the reference: the signs of zero updates follow IEEE as in adamw_update
    (optimizer.cpp:57-68), zero moments pack to +0 (expand.cpp:18-22)."""
    import torch
    n = 128 * 96
    r = rng(71)
    w0 = (r.standard_normal(n) * 0.02).astype(np.float32)
    w0[::7] = 0.0
    w0[3::7] = -0.0
    w0[128 * 5:128 * 6] = -0.0
    m, v = checker.make_slot(n)
    slot = coat.make_slot([n])
    w_ref, w = w0.copy(), dev(w0)
    c = coat.AdamWConfig(**CFG)
    for t in range(3):
        g = (r.standard_normal(n) * 1e-3).astype(np.float32)
        g[::5] = -0.0
        g[2::5] = 0.0
        g[128 * 7:128 * 9] = -0.0
        assert checker.step(w_ref, g, m, v, t, CFG) == 0
        coat.step(w, dev(g), slot, c)
        wd = host(w)
        bad = np.nonzero(wd.view(np.uint32) != w_ref.view(np.uint32))[0]
        assert bad.size == 0, (t, bad[:8], wd[bad[:8]], w_ref[bad[:8]])
        gm, gv = gpu_state(slot)
        assert_state_equal(gm, m, f"m step {t}")
        assert_state_equal(gv, v, f"v step {t}")


def test_step_subnormal_moment_groups(coat, port, checker):
    """Gradients ~1e-21 make v' = (1 - b2) g^2 subnormal; such a group's
    c = sqrt(lo * hi) is subnormal too, and with k > 1 the expanded maximum
    must come from pow(hi / (double)c, k) as in the reference (a float
    RN(1/c) overflows).  Found by tests/test_gpu_fuzz.py."""
    r = rng(81)
    n = 128 * 64
    w0 = (r.standard_normal(n) * 0.02).astype(np.float32)
    g = (r.standard_normal(n) * 1e-3).astype(np.float32)
    for q in range(0, 64, 3):   # every third group: subnormal v', mixed with zeros
        gg = (r.standard_normal(128) * 10.0 ** r.uniform(-22.5, -21)).astype(np.float32)
        gg[r.random(128) < 0.3] = 0.0
        g[q * 128:(q + 1) * 128] = gg
    m, v = checker.make_slot(n)
    w_ref = w0.copy()
    assert checker.step(w_ref, g, m, v, 0, CFG) == 0
    assert (v["k"] > 1).any() and (v["c"] < 2.0 ** -126).any()   # the case is exercised
    slot = coat.make_slot([n])
    w = dev(w0)
    coat.step(w, dev(g), slot, coat.AdamWConfig(**CFG))
    assert np.array_equal(host(w).view(np.uint32), w_ref.view(np.uint32))
    gm, gv = gpu_state(slot)
    assert_state_equal(gm, m, "m")
    assert_state_equal(gv, v, "v")
