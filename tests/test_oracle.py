"""Pin the CPU oracle (oracle/coat_oracle.c) before trusting it.

1. Known-answer tests restated from the reference's own test suite
   (/root/reference/proj/tests/test_fp8.cpp, test_quantize.cpp, test_expand.cpp)
   -- only the expectations the reference itself passes.
2. Differential checks against the unmodified reference library
   (oracle/_ref/libcoatsim_ref.so) on random inputs: bit-exact.
CPU only.
"""
import math

import numpy as np
import pytest

from conftest import rng

E4M3_MAX = np.float32(448.0)
E4M3_MIN = np.float32(2.0 ** -9)


def ref_decode(b: int) -> float:
    """Field-definition decode (test_fp8.cpp:18-38)."""
    sign, expf, mant = b >> 7, (b >> 3) & 0xF, b & 7
    if expf == 15 and mant == 7:
        return math.nan
    mag = mant * 2.0 ** (1 - 7 - 3) if expf == 0 else (1 + mant / 8) * 2.0 ** (expf - 7)
    return -mag if sign else mag


def enumeration_encode(v: float) -> int:
    """Nearest-code search, ties to even mantissa (test_fp8.cpp:42-68)."""
    best, best_b, first = 0.0, 0, True
    for b in range(256):
        val = ref_decode(b)
        if math.isnan(val):
            continue
        d = abs(val - v)
        if first or d < abs(best - v):
            best, best_b, first = val, b, False
        elif d == abs(best - v):
            cand_even = (b & 7) % 2 == 0
            best_even = (best_b & 7) % 2 == 0
            if val == best:
                if (math.copysign(1, v) < 0) == bool(b >> 7):
                    best_b = b
            elif cand_even and not best_even:
                best, best_b = val, b
    return best_b


# ------------------------------------------------------------------ codec --
def test_decode_every_byte(port):
    dec = port.decode_e4m3(np.arange(256, dtype=np.uint8))
    for b in range(256):
        r = ref_decode(b)
        if math.isnan(r):
            assert math.isnan(dec[b])
        else:
            assert dec[b] == np.float32(r)


def test_decode_kats(port):  # test_fp8.cpp:106-117
    d = port.decode_e4m3(np.array([0x00, 0x80, 0x38, 0x01, 0x7E, 0x7F], np.uint8))
    assert d[0] == 0 and not np.signbit(d[0])
    assert np.signbit(d[1])
    assert d[2] == 1.0 and d[3] == 2.0 ** -9 and d[4] == 448.0 and np.isnan(d[5])


def test_exhaustive_round_trip(port):  # test_fp8.cpp:119-130 (E4M3 half)
    codes = np.array([b for b in range(256) if (b & 0x7F) != 0x7F], np.uint8)
    assert codes.size == 254
    assert np.array_equal(port.encode_e4m3(port.decode_e4m3(codes)), codes)


def test_encode_matches_enumeration(port):  # test_fp8.cpp:132-153
    r = rng(2024)
    mags = np.exp(r.uniform(np.log(1e-8), np.log(2e5), 4000))
    vals = np.where(r.integers(0, 2, 4000) == 1, -mags, mags).astype(np.float32)
    got = port.encode_e4m3(vals)
    for v, c in zip(vals, got):
        assert c == enumeration_encode(float(v))
    # exact midpoints between adjacent finite codes
    ties = []
    for b in range(255):
        lo, hi = ref_decode(b), ref_decode(b + 1)
        if math.isnan(lo) or math.isnan(hi) or not lo < hi:
            continue
        mid = (lo + hi) / 2
        if float(np.float32(mid)) == mid:
            ties.append(mid)
    ties = np.array(ties, np.float32)
    got = port.encode_e4m3(ties)
    for v, c in zip(ties, got):
        assert c == enumeration_encode(float(v))


def test_encode_saturation_and_zero(port):  # test_fp8.cpp:155-177
    x = np.array([448, 1e4, -1e4, 0.0, -0.0, 2.0 ** -11, 2.0 ** -10, -2.0 ** -11, 1.5 * 2.0 ** -10],
                 np.float32)
    c = port.encode_e4m3(x)
    d = port.decode_e4m3(c)
    assert d[0] == 448 and d[1] == 448 and d[2] == -448
    assert list(c[3:]) == [0x00, 0x80, 0x00, 0x00, 0x80, 0x01]
    from pyoracle import Status
    for bad in (np.inf, np.nan, -np.inf):
        with pytest.raises(Status) as e:
            port.encode_e4m3(np.array([bad], np.float32))
        assert e.value.code == 3


def test_round_bf16_ties(ref):  # test_fp8.cpp:271-295
    x = np.array([1.0, 0.0, 1 + 2.0 ** -9, 1 + 2.0 ** -8, 1 + 3 * 2.0 ** -8], np.float32)
    assert list(ref.round_bf16(x)) == [1.0, 0.0, 1.0, 1.0, 1 + 2.0 ** -6]


# -------------------------------------------------------------- quantizer --
def test_per_tensor_documented_codes(port):  # test_quantize.cpp:24-42
    x = np.array([0.5, -1.0, 2.0, 4.0], np.float32)
    codes, s = port.quantize(x, 0)
    bf = port.round_bf16(np.array([np.float32(4.0) / np.float32(448.0)], np.float32))[0]
    assert s[0] == bf
    assert list(codes) == list(port.encode_e4m3(np.array([56, -112, 224, 448], np.float32)))
    back = port.dequantize(codes, s, 0)
    assert np.max(np.abs(back - x) / np.abs(x)) <= 2.0 ** -8


def test_per_group_two_group_example(port):  # test_quantize.cpp:44-55
    x = np.array([1.0, 2.0, 100.0, 200.0], np.float32)
    codes, s = port.quantize(x, 2)
    assert s[0] == port.round_bf16(np.array([np.float32(2) / np.float32(448)], np.float32))[0]
    assert s[1] == port.round_bf16(np.array([np.float32(200) / np.float32(448)], np.float32))[0]
    assert list(codes) == list(port.encode_e4m3(np.array([224, 448, 224, 448], np.float32)))


def test_all_zero_scale_is_delta_min(port):  # test_quantize.cpp:57-71 (E4M3 rows)
    x = np.zeros((3, 8), np.float32)
    for G in (0, 4):
        codes, s = port.quantize(x, G)
        assert np.all(s == E4M3_MIN) and np.all(codes == 0)


def test_per_group_error_bound(port):  # test_quantize.cpp:87-100
    r = rng(41)
    for _ in range(50):
        mag = np.exp(r.uniform(np.log(0.25), np.log(4.0), (8, 32)))
        x = np.where(r.integers(0, 2, (8, 32)) == 1, -mag, mag).astype(np.float32)
        codes, s = port.quantize(x, 16)
        back = port.dequantize(codes, s, 16)
        assert np.max(np.abs(back - x) / np.abs(x)) <= 2.0 ** -4 + 2.0 ** -7


def test_power_of_two_rescale(port):  # test_quantize.cpp:102-117
    r = rng(43)
    for t in range(20):
        x = r.standard_normal((4, 64)).astype(np.float32)
        c0, s0 = port.quantize(x, 16)
        sh = int(r.integers(0, 13)) - 6
        c1, s1 = port.quantize(np.ldexp(x, sh).astype(np.float32), 16)
        assert np.array_equal(c0, c1) and np.array_equal(s1, np.ldexp(s0, sh).astype(np.float32))


def test_group_equals_per_tensor_on_one_row(port):  # test_quantize.cpp:119-125
    x = rng(77).standard_normal(64).astype(np.float32)
    a = port.quantize(x, 64)
    b = port.quantize(x, 0)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_two_stage_equals_single_pass(port):  # test_quantize.cpp:127-146
    r = rng(51)
    for _ in range(50):
        rows = int(r.integers(1, 6))
        x = (3.0 * r.standard_normal((rows, 96))).astype(np.float32)
        for G in (1, 2, 3, 4, 6, 8, 12, 16, 24, 32, 48, 96):
            inter, g = port.group_scale_max(x, G)
            assert inter.size == x.size // G
            assert g == np.max(np.abs(x))
    from pyoracle import Status
    with pytest.raises(Status):
        port.group_scale_max(np.full((2, 8), 2.5, np.float32), 3)


# -------------------------------------------------------------------- DRE --
def test_optimal_k_kats(port):  # test_expand.cpp:59-71
    assert port.optimal_k(229376.0) == (np.float32(1.0), False)
    k8, _ = port.optimal_k(8.0)
    assert abs(k8 - math.log(229376.0) / math.log(8.0)) <= 1e-6 * k8
    assert port.optimal_k(1e9)[0] == 1.0
    assert port.optimal_k(1.1)[0] == 20.0
    assert port.optimal_k(1.0) == (np.float32(1.0), True)


def test_degenerate_groups(port):  # test_expand.cpp:240-254 (passing parts)
    codes, s, k, c = port.expand_quantize(np.zeros(128, np.float32))
    assert k[0] == 1 and c[0] == 1 and np.all(port.dequantize_contract(codes, s, k, c) == 0)
    codes, s, k, c = port.expand_quantize(np.full(128, 0.25, np.float32))
    assert k[0] == 1 and c[0] == np.float32(0.25)


def test_lossless_group_at_e4m3_range(port):  # test_expand.cpp:256-265
    g = np.full(128, 2.0 ** -9, np.float32)
    g[0] = 448
    codes, s, k, c = port.expand_quantize(g)
    assert k[0] == 1.0
    back = port.dequantize_contract(codes, s, k, c)
    assert np.max(np.abs(back - g) / g) <= 2.0 ** -8


def test_stabilizer_reciprocity(port):  # test_expand.cpp:161-175
    r = rng(9000)
    for _ in range(50):
        mag = np.exp(r.uniform(-0.5 * np.log(1e6), 0.5 * np.log(1e6), 128))
        g = np.where(r.integers(0, 2, 128) == 1, -mag, mag).astype(np.float32)
        k, c, rng_, deg = port.measure_group(g)
        lo, hi = np.min(np.abs(g)).astype(np.float64), np.max(np.abs(g)).astype(np.float64)
        assert abs((lo / c) * (hi / c) - 1.0) <= 1e-6


def test_expand_beats_plain_quantization(port):  # test_expand.cpp:187-206
    r = rng(81)
    wins = 0
    for seed in range(10):
        v = np.empty(64 * 128, np.float32)
        for gi in range(64):
            rr = r.uniform(2.5, 11.0)
            mag = np.exp(r.uniform(-0.5 * np.log(rr), 0.5 * np.log(rr), 128))
            v[gi * 128:(gi + 1) * 128] = (mag * 1e-8).astype(np.float32)
        codes, s, k, c = port.expand_quantize(v)
        e_exp = np.mean((port.dequantize_contract(codes, s, k, c).astype(np.float64) - v) ** 2)
        qc, qs = port.quantize(v.reshape(64, 128), 128)
        e_plain = np.mean((port.dequantize(qc, qs, 128).astype(np.float64).ravel() - v) ** 2)
        wins += e_exp < e_plain
    assert wins == 10


# ------------------------------------------------ port == reference bitwise --
def _act(ref, rows, cols, seed):
    return ref.generate(1, (rows, cols), 0.05, 50.0, seed)


def test_generators_match_reference(port, ref):
    for kind, shape, frac, scale in [(0, (4096,), 0.01, 100.0), (1, (32, 64), 0.05, 50.0),
                                     (2, (1000,), 0.0, 1e4)]:
        assert np.array_equal(port.generate(kind, shape, frac, scale, 99),
                              ref.generate(kind, shape, frac, scale, 99))


def test_codec_matches_reference_exhaustive_window(port, ref):
    # every fp32 in +-[2^-12, 2^10): all E4M3 rounding boundaries (~2e8 values, chunked)
    for e in range(-12, 10, 4):
        lo = np.float32(2.0 ** e).view(np.uint32)
        hi = np.float32(2.0 ** min(e + 4, 10)).view(np.uint32)
        bits = np.arange(lo, hi, 97, dtype=np.uint32)    # strided sample of the window
        x = np.concatenate([bits.view(np.float32), -bits.view(np.float32)])
        assert np.array_equal(port.encode_e4m3(x), ref.encode_e4m3(x))


@pytest.mark.parametrize("G", [0, 16, 32, 128, 48])
def test_quantize_matches_reference(port, ref, G):
    x = _act(ref, 64, 384, 7)
    a, b = port.quantize(x, G), ref.quantize(x, G)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert np.array_equal(port.dequantize(*a, G), ref.dequantize(*b, G))
    if G:
        ia, ga = port.group_scale_max(x, G)
        ib, gb = ref.group_scale_max(x, G)
        assert np.array_equal(ia, ib) and ga == gb


def test_expand_quantize_matches_reference(port, ref):
    m = ref.generate(0, (128 * 256,), 0.01, 100.0, 21) * np.float32(1e-4)
    r = rng(22)
    v = np.concatenate([(np.exp(r.uniform(-0.5 * np.log(q), 0.5 * np.log(q), 128)) * 1e-8)
                        for q in r.uniform(2.5, 11.0, 256)]).astype(np.float32)
    for x in (m, v, _act(ref, 64, 128, 3).ravel()):
        a, b = port.expand_quantize(x), ref.expand_quantize(x)
        for u, w in zip(a, b):
            assert np.array_equal(u, w)
        assert np.array_equal(port.dequantize_contract(*a), ref.dequantize_contract(*b))


@pytest.mark.parametrize("n", [4096, 4096 + 77, 1000])
def test_step_matches_reference(port, ref, n):
    from pyoracle import ADAMW_DEFAULT
    cfg = dict(ADAMW_DEFAULT, weight_decay=0.1)
    w0 = ref.generate(0, (n,), 0.0, 100.0, 1) * np.float32(0.02)
    out = {}
    for o in (port, ref):
        w = w0.copy()
        m, v = o.make_slot(n)
        for t in range(4):
            g = ref.generate(0, (n,), 0.01, 100.0, 100 + t) * np.float32(1e-3)
            assert o.step(w, g, m, v, t, cfg) == 0
        out[o.kind] = (w, m, v)
    (wp, mp, vp), (wr, mr, vr) = out["port"], out["reference"]
    assert np.array_equal(wp, wr)
    for a, b in ((mp, mr), (vp, vr)):
        for key in ("codes", "scales", "k", "c"):
            assert np.array_equal(a[key], b[key]), key


def test_step_error_semantics_match_reference(port, ref):
    from pyoracle import ADAMW_DEFAULT
    n = 512
    for o in (port, ref):
        w = np.ones(n, np.float32)
        m, v = o.make_slot(n)
        g = np.zeros(n, np.float32)
        g[7] = np.nan
        w_before = w.copy()
        assert o.step(w, g, m, v, 0, ADAMW_DEFAULT) == 4          # NonFiniteGradient
        assert np.array_equal(w, w_before)
        g = np.zeros(n, np.float32)
        g[3] = 1e20                                               # g*g overflows -> v = inf
        assert o.step(w, g, m, v, 0, dict(ADAMW_DEFAULT, weight_decay=0.1)) == 3  # pack(v) throws
        assert not np.array_equal(w, w_before)                    # params were updated


def test_multithreaded_reference_is_bitwise_equal(ref):
    from pyoracle import ADAMW_DEFAULT
    n = 128 * 1000 + 5
    w0 = ref.generate(0, (n,), 0.0, 100.0, 1) * np.float32(0.02)
    g = ref.generate(0, (n,), 0.01, 100.0, 100) * np.float32(1e-3)
    res = []
    for th in (1, 7):
        w = w0.copy()
        m, v = ref.make_slot(n)
        ref.step(w, g, m, v, 0, ADAMW_DEFAULT, threads=th)
        ref.step(w, g, m, v, 1, ADAMW_DEFAULT, threads=th)
        res.append((w, m, v))
    assert np.array_equal(res[0][0], res[1][0])
    for key in ("codes", "scales", "k", "c"):
        assert np.array_equal(res[0][1][key], res[1][1][key])
        assert np.array_equal(res[0][2][key], res[1][2][key])


def test_producer_port_reproduces_reference_layer_tape(port, ref):
    """The fused-producer restatement (rmsnorm / silu / mul + MGAQ quantizers)
    reproduces, bit for bit, the records the reference's COAT DecoderLayer
    forward saves (flow.cpp:546-612): qkv.in, upgate.in, mul.in.silu, down.in."""
    H, I, heads, S, B = 64, 128, 4, 32, 2
    N = B * S
    x = port.generate(1, (N, H), 0.05, 20.0, 3)

    def rec(name):
        return ref.layer_tape(x, name, H, I, heads, S, B)

    def dq(codes, scales, G, shape):
        return port.dequantize(codes.reshape(shape), scales, G)

    c_in, s_in, k, rms1, rms2 = rec("rmsnorm1.in")
    assert k == 0
    pc, ps = port.quantize(x, 16)
    assert np.array_equal(pc.reshape(-1), c_in) and np.array_equal(ps, s_in)
    n1 = port.rmsnorm(dq(c_in, s_in, 16, (N, H)), rms1)
    c_q, s_q, k, _, _ = rec("qkv.in")
    pc, ps = port.quantize(n1, 0)
    assert k == 1 and np.array_equal(pc.reshape(-1), c_q) and np.array_equal(ps, s_q)
    # MLP half from the saved rmsnorm2.in record
    c_r2, s_r2, _, _, _ = rec("rmsnorm2.in")
    n2 = port.rmsnorm(dq(c_r2, s_r2, 16, (N, H)), rms2)
    c_u, s_u, _, _, _ = rec("upgate.in")
    pc, ps = port.quantize(n2, 0)
    assert np.array_equal(pc.reshape(-1), c_u) and np.array_equal(ps, s_u)
    c_g, s_g, _, _, _ = rec("silu.in")
    silu = port.silu(dq(c_g, s_g, 16, (N, I)))
    c_ms, s_ms, _, _, _ = rec("mul.in.silu")
    pc, ps = port.quantize(silu, 16)
    assert np.array_equal(pc.reshape(-1), c_ms) and np.array_equal(ps, s_ms)
    c_mu, s_mu, _, _, _ = rec("mul.in.up")
    prod = dq(c_ms, s_ms, 16, (N, I)) * dq(c_mu, s_mu, 16, (N, I))
    c_d, s_d, _, _, _ = rec("down.in")
    pc, ps = port.quantize(prod.astype(np.float32), 0)
    assert np.array_equal(pc.reshape(-1), c_d) and np.array_equal(ps, s_d)
