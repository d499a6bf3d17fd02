"""Backward-side MGAQ pieces vs the oracle, bit-exact:
used_values_transposed (flow.cpp:360-395), requantize_cached (flow.cpp:487-495)
and the per-cycle weight-scale cache (flow.cpp:499-530)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("rows,cols,G", [(100, 256, 16), (64, 4096, 0), (333, 128, 128), (7, 48, 16),
                                         (8192, 4096, 0), (8192, 5120, 0), (8192, 11008, 16)])   # full sizes
@pytest.mark.parametrize("odt", ["fp32", "bf16"])
def test_used_values_transposed(coat, port, rows, cols, G, odt):
    import torch
    x = port.generate(1, (rows, cols), 0.05, 30.0, 4)
    q = coat.quantize(torch.from_numpy(x).cuda(), coat.QuantGeometry.per_group(G) if G else
                      coat.QuantGeometry.per_tensor())
    out_dtype = torch.float32 if odt == "fp32" else torch.bfloat16
    t, ct = coat.used_values_transposed(q, out_dtype, return_codes=True)
    codes, scales = port.quantize(x, G)
    ref = port.dequantize(codes, scales, G).T.copy()
    assert np.array_equal(ct.cpu().numpy(), codes.T)
    got = t.float().cpu().numpy()
    if odt == "bf16":   # round_bf16 (fp8.cpp:209-216) == torch's RNE bf16 cast for finite values
        ref = torch.from_numpy(ref).to(torch.bfloat16).float().numpy()
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))


@pytest.mark.parametrize("n", [8192 * 64, 1000 * 16 + 7, 8192 * 4096])   # the last: attn.out at full size
def test_requantize_cached(coat, port, n):
    import torch
    x = port.generate(1, (n,), 0.05, 30.0, 6)
    x[5] = -0.0
    xb = torch.from_numpy(x).to(torch.bfloat16)
    xf = xb.float().numpy()
    q = coat.quantize(xb.cuda(), coat.QuantGeometry.per_tensor())
    s = q.scales.float().cpu().numpy()[0]
    out, codes = coat.requantize_cached(xb.cuda(), q.scales, return_codes=True)
    exp_codes = port.encode_e4m3((xf / np.float32(s)).astype(np.float32))
    assert np.array_equal(codes.cpu().numpy(), exp_codes)
    assert np.array_equal(codes.cpu().numpy(), q.codes.cpu().numpy())     # == the forward's codes
    exp = (port.decode_e4m3(exp_codes) * np.float32(s)).astype(np.float32)
    assert np.array_equal(out.cpu().numpy().view(np.uint32), exp.view(np.uint32))


def test_weight_operand_cache(coat):
    import torch
    cache = coat.WeightOperandCache()
    w = torch.randn(256, 512, device="cuda")
    a = cache.operand("wq", w)
    b = cache.operand("wq", w * 2)          # same cycle: cached operand, no new scale
    assert a is b and cache.weight_scale_computations == 1
    cache.start_accumulation_cycle()
    c = cache.operand("wq", w * 2)
    assert cache.weight_scale_computations == 2
    assert not torch.equal(a.scales, c.scales)
