"""GPU: the SiLU producer's paired expf (coat_device.cuh expf_neg2: CUDA's
expf instruction sequence issued as FFMA2 / FADD2 / FMUL2) equals CUDA's scalar
expf(-x) bit for bit on every float (2^32 inputs, NaNs and infinities
included).  silu = x * RN(1 / RN(1 + expf(-x))) (flow.cpp:97-104)."""
import pytest

pytestmark = pytest.mark.gpu


def test_expf_neg2_exhaustive(coat):
    import torch
    from paper_2410_19313_b200 import _lib
    bad = torch.zeros(1, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    assert _lib.lib.coat_test_expf_neg2(0, 1 << 32, bad.data_ptr(), st) == 0
    torch.cuda.synchronize()
    assert int(bad.item()) == 0
