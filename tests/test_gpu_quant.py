"""GPU parity: E4M3 codec and MGAQ quantizers (K2/K3) vs the CPU oracle, bit-exact.

Reference: fp8.cpp:27-156, quantize.cpp:89-145; call sites flow.cpp:450-480.
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
    if t.dtype == torch.bfloat16:
        return t.float().cpu().numpy()
    return t.cpu().numpy()


def bf16_round_np(x):
    u = x.astype(np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def test_encode_exhaustive_window(coat, port):
    """Every fp32 bit pattern with |x| in [2^-12, 2^10) (all E4M3 rounding
    boundaries), both signs, plus specials: GPU cvt == encode_byte."""
    lo = np.float32(2.0 ** -12).view(np.uint32)
    hi = np.float32(2.0 ** 10).view(np.uint32)
    step = 1 << 24
    for b0 in range(int(lo), int(hi), step):
        bits = np.arange(b0, min(b0 + step, int(hi)), dtype=np.uint32)
        x = bits.view(np.float32)
        for sgn in (1, -1):
            xs = (x * np.float32(sgn)).astype(np.float32)
            got = host(coat.encode_e4m3(dev(xs)))
            assert np.array_equal(got, port.encode_e4m3(xs))
    # tails: zeros, fp32 subnormals, huge values, every decoded value
    special = np.concatenate([
        np.array([0.0, -0.0, 1e-45, -1e-45, 1e-40, 3e38, -3e38, 448, 464, 465, -464, 480], np.float32),
        port.decode_e4m3(np.array([b for b in range(256) if b & 0x7F != 0x7F], np.uint8))])
    assert np.array_equal(host(coat.encode_e4m3(dev(special))), port.encode_e4m3(special))


def test_decode_all_codes(coat, port):
    codes = np.arange(256, dtype=np.uint8)
    got = host(coat.decode_e4m3(dev(codes)))
    exp = port.decode_e4m3(codes)
    assert np.array_equal(np.isnan(got), np.isnan(exp))
    ok = ~np.isnan(exp)
    assert np.array_equal(got[ok].view(np.uint32), exp[ok].view(np.uint32))


def test_encode_nonfinite_raises(coat):
    for bad in (np.inf, np.nan):
        with pytest.raises(coat.NonFiniteInput):
            coat.encode_e4m3(dev(np.array([1.0, bad], np.float32)))


def _activation(ref_or_port, rows, cols, seed, frac=0.01, scale=50.0):
    return ref_or_port.generate(1, (rows, cols), frac, scale, seed)


@pytest.mark.parametrize("G", [16, 32, 64, 128, 256, 512, 48, 8])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_quantize_per_group_bit_exact(coat, port, G, dtype):
    import torch
    x = _activation(port, 96, 1536, 11 + G)
    if dtype == "bf16":
        x = bf16_round_np(x)   # bf16 device input == fp32 oracle input
    xt = dev(x) if dtype == "f32" else dev(x).to(torch.bfloat16)
    q = coat.quantize(xt, coat.QuantGeometry.per_group(G))
    codes, scales = port.quantize(x, G)
    assert np.array_equal(host(q.codes), codes)
    assert np.array_equal(host(q.scales), scales)
    back = coat.dequantize(q)
    assert np.array_equal(host(back), port.dequantize(codes, scales, G))


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("shape", [(64, 4096), (33, 384), (7, 100), (1, 64)])
def test_quantize_per_tensor_bit_exact(coat, port, dtype, shape):
    import torch
    x = _activation(port, shape[0], shape[1], 5)
    if dtype == "bf16":
        x = bf16_round_np(x)
    xt = dev(x) if dtype == "f32" else dev(x).to(torch.bfloat16)
    q = coat.quantize(xt, coat.QuantGeometry.per_tensor())
    codes, scales = port.quantize(x, 0)
    assert np.array_equal(host(q.codes), codes)
    assert host(q.scales)[0] == scales[0]
    assert np.array_equal(host(coat.dequantize(q)), port.dequantize(codes, scales, 0))


@pytest.mark.parametrize("G", [1, 3, 16, 128, 96])
def test_group_scale_max_two_stage(coat, port, G):
    x = (3.0 * rng(51 + G).standard_normal((5, 384))).astype(np.float32)
    inter, g = coat.group_scale_max(dev(x), G)
    pi, pg = port.group_scale_max(x, G)
    assert np.array_equal(host(inter), pi) and np.float32(g) == pg == np.max(np.abs(x))


def test_quantizer_kats(coat, port):
    # test_quantize.cpp:24-71
    q = coat.quantize(dev(np.array([[0.5, -1.0, 2.0, 4.0]], np.float32)), coat.QuantGeometry.per_tensor())
    assert list(host(q.codes).ravel()) == list(port.encode_e4m3(np.array([56, -112, 224, 448], np.float32)))
    q = coat.quantize(dev(np.array([[1.0, 2.0, 100.0, 200.0]], np.float32)), coat.QuantGeometry.per_group(2))
    assert list(host(q.codes).ravel()) == list(port.encode_e4m3(np.array([224, 448, 224, 448], np.float32)))
    for geo in (coat.QuantGeometry.per_tensor(), coat.QuantGeometry.per_group(4)):
        q = coat.quantize(dev(np.zeros((3, 8), np.float32)), geo)
        assert np.all(host(q.scales) == 2.0 ** -9) and np.all(host(q.codes) == 0)


def test_quantizer_errors(coat):
    x = dev(np.zeros((4, 6), np.float32))
    with pytest.raises(coat.GeometryMismatch):
        coat.quantize(x, coat.QuantGeometry.per_group(5))
    with pytest.raises(coat.InvalidSpec):
        coat.quantize(x, coat.QuantGeometry.per_block(2))
    y = np.ones((4, 64), np.float32)
    y[2, 5] = np.nan
    for geo in (coat.QuantGeometry.per_tensor(), coat.QuantGeometry.per_group(16)):
        with pytest.raises(coat.NonFiniteInput):
            coat.quantize(dev(y), geo)


def test_power_of_two_rescale_gpu(coat):
    r = rng(43)
    for _ in range(10):
        x = r.standard_normal((4, 64)).astype(np.float32)
        sh = int(r.integers(0, 13)) - 6
        a = coat.quantize(dev(x), coat.QuantGeometry.per_group(16))
        b = coat.quantize(dev(np.ldexp(x, sh).astype(np.float32)), coat.QuantGeometry.per_group(16))
        assert np.array_equal(host(a.codes), host(b.codes))
        assert np.array_equal(host(b.scales), np.ldexp(host(a.scales), sh))


def test_llama_layer_sizes_bit_exact_full(coat, port):
    """Config-2 shapes at full size (8192 x 11008 bf16, 90M elements): every
    code and scale of the per-group (1x16) quantization against the oracle, and
    the per-tensor (Group Scaling) scale plus every code of it."""
    import torch
    rows, cols = 8192, 11008
    g = torch.Generator(device="cuda").manual_seed(3)
    xt = (torch.randn(rows, cols, device="cuda", generator=g) * 3).to(torch.bfloat16)
    xt[5] *= 50
    xt[::97, ::13] = 0.0
    q = coat.quantize(xt, coat.QuantGeometry.per_group(16))
    sample = list(range(rows))
    xs = xt[sample].float().cpu().numpy()
    codes, scales = port.quantize(xs, 16)
    assert np.array_equal(host(q.codes[sample]), codes)
    assert np.array_equal(host(q.scales.view(rows, cols // 16)[sample]).ravel(), scales)
    qt = coat.quantize(xt, coat.QuantGeometry.per_tensor())
    amax = float(xt.float().abs().max())
    s = bf16_round_np(np.array([np.float32(amax) / np.float32(448.0)], np.float32))[0]
    assert host(qt.scales)[0] == s
    exp = port.encode_e4m3((xs / s).astype(np.float32)).reshape(xs.shape)
    assert np.array_equal(host(qt.codes[sample]), exp)


@pytest.mark.parametrize("mode", ["coop", "queue"])
def test_quantize_batch_alternate_schedules_match_single_calls(mode):
    """The single cooperative launch (COAT_MGAQ_BATCH=coop) and the persistent
    warp-specialised task-queue kernel (=queue) behind coat_quantize_batch --
    chosen once per process, hence a subprocess -- give the entry points'
    results too, incl. the full Llama-2-7B layer."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, COAT_MGAQ_BATCH=mode)
    here = os.path.dirname(os.path.abspath(__file__))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.join(here, "test_gpu_quant.py"), "-k", "batch and not alternate"],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "passed" in r.stdout


def test_quantize_batch_llama_layer_matches_single_calls(coat):
    """The nine MGAQ records of a Llama-2-7B layer (cfg2: 8192 tokens, H 4096,
    I 11008; per-group 1x16 and per-tensor) in one coat_quantize_batch call,
    bit-identical to the per-tensor entry points record by record."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(21)
    specs = [((8192, 4096), 16), ((8192, 4096), 0), ((8192, 4096), 0), ((8192, 4096), 16), ((8192, 4096), 0),
             ((8192, 11008), 16), ((8192, 11008), 16), ((8192, 11008), 16), ((8192, 11008), 0)]
    xs = []
    for shape, G in specs:
        x = torch.randn(shape, device="cuda", generator=g) * 2
        x[::100] *= 50
        xs.append((x.to(torch.bfloat16), coat.QuantGeometry.per_group(G) if G else coat.QuantGeometry.per_tensor()))
    batch = coat.quantize_batch(xs)
    for (x, geo), qb in zip(xs, batch):
        q = coat.quantize(x, geo)
        assert torch.equal(q.codes, qb.codes)
        assert torch.equal(q.scales.view(torch.int16), qb.scales.view(torch.int16))


def test_quantize_batch_matches_single_calls(coat):
    """coat_quantize_batch (a layer's MGAQ records in one call: 3 internal
    streams by default) is bit-identical to the per-tensor entry points, mixed
    geometries and dtypes."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(3)
    specs = [((96, 256), torch.bfloat16, coat.QuantGeometry.per_group(16)),
             ((64, 512), torch.bfloat16, coat.QuantGeometry.per_tensor()),
             ((33, 128), torch.float32, coat.QuantGeometry.per_group(128)),
             ((40, 384), torch.float32, coat.QuantGeometry.per_tensor()),
             ((7, 4096), torch.bfloat16, coat.QuantGeometry.per_group(32)),
             ((129, 1024), torch.bfloat16, coat.QuantGeometry.per_tensor())]
    xs = []
    for shape, dt, geo in specs:
        x = torch.randn(shape, device="cuda", generator=g) * 3
        x[::17] *= 300
        x[1, :5] = 0
        xs.append((x.to(dt), geo))
    batch = coat.quantize_batch(xs)
    for (x, geo), qb in zip(xs, batch):
        q = coat.quantize(x, geo)
        assert torch.equal(q.codes, qb.codes)
        assert torch.equal(q.scales.view(torch.int16), qb.scales.view(torch.int16))


def test_quantize_batch_nonfinite_raises(coat):
    import torch
    x = torch.randn(64, 256, device="cuda").to(torch.bfloat16)
    y = torch.randn(64, 256, device="cuda").to(torch.bfloat16)
    y[5, 7] = float("inf")
    with pytest.raises(coat.NonFiniteInput):
        coat.quantize_batch([(x, coat.QuantGeometry.per_group(16)), (y, coat.QuantGeometry.per_tensor())])


@pytest.mark.parametrize("geo_g", [16, 128, 0])
@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_signed_zero_inputs_encode_like_reference(coat, port, geo_g, dtype):
    """encode_byte(-0) = 0x80 (fp8.cpp:53-88): -0 inputs keep their sign bit
    through the exact (Markstein) quotient."""
    import torch
    x = port.generate(1, (32, 256), 0.05, 10.0, 5)
    x[3, :40] = -0.0
    x[4, 7] = 0.0
    x[5, :] = -0.0          # an all -0 group row
    xt = torch.from_numpy(x).cuda()
    if dtype == "bf16":
        xt = xt.to(torch.bfloat16)
        x = xt.float().cpu().numpy()
    geo = coat.QuantGeometry.per_group(geo_g) if geo_g else coat.QuantGeometry.per_tensor()
    q = coat.quantize(xt, geo)
    codes, scales = port.quantize(x, geo_g)
    assert np.array_equal(q.codes.cpu().numpy(), codes)
    assert np.array_equal(q.scales.float().cpu().numpy(), scales)
    qb = coat.quantize_batch([(xt, geo)])[0]
    assert np.array_equal(qb.codes.cpu().numpy(), codes)


@pytest.mark.parametrize("n", [256, 4099, 1 << 20])
def test_decode_e4m3_bf16_exact(coat, n):
    """coat_decode_e4m3_bf16 (the BF16 code values for the backward GEMMs): the
    vectorized 16-codes-per-thread kernel and the scalar tail give exactly the
    top half of the fp32 decode (<= 4 significant bits: exact in BF16); NaN
    codes decode to a NaN."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(n)
    codes = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda", generator=g)
    codes[:256] = torch.arange(256, dtype=torch.uint8, device="cuda")
    out = coat.decode_e4m3_bf16(codes)
    ref = coat.decode_e4m3(codes)
    torch.cuda.synchronize()
    nan = torch.isnan(ref)
    assert bool(torch.isnan(out.float())[nan].all())
    got = out.view(torch.int16)[~nan]
    want = (ref.view(torch.int32)[~nan] >> 16).to(torch.int16)
    assert torch.equal(got, want)
