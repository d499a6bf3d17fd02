"""GPU: the host-buffer step (coat_adamw_dre_step_host, the path bench.py's
e2e number uses: params and grads in pinned host memory streamed through the
GPU in chunks, state resident in HBM) equals the device-buffer step
(coat_adamw_dre_step) bit for bit -- weights and state -- with chunks that do
not divide n (ragged last chunk) over several steps.  optimizer.cpp:101-114.
"""
import ctypes as C

import numpy as np
import pytest

from conftest import rng

pytestmark = pytest.mark.gpu

CFG = {"beta1": 0.9, "beta2": 0.999, "lr": 1e-3, "weight_decay": 0.1, "eps": 1e-8}


@pytest.mark.parametrize("n,chunk", [(1792 * 300 + 128 * 3, 50_000), (128 * 10, 1 << 20), (1 << 20, 1792)])
def test_host_step_equals_device_step(n, chunk):
    import torch
    from paper_2410_19313_b200 import _lib
    L = _lib.lib
    ng = -(-n // 128)

    def moment():
        return {"codes": torch.zeros(n, dtype=torch.uint8, device="cuda"),
                "scales": torch.full((ng,), 0x3B00, dtype=torch.int16, device="cuda"),
                "k": torch.ones(ng, device="cuda"), "c": torch.ones(ng, device="cuda")}

    def cs(mm):
        return _lib.MomentState(mm["codes"].data_ptr(), mm["scales"].data_ptr(), mm["k"].data_ptr(),
                                mm["c"].data_ptr())

    r = rng(61)
    w0 = (r.standard_normal(n) * 0.02).astype(np.float32)
    cfg = _lib.AdamWConfigC(**CFG)
    st = torch.cuda.current_stream().cuda_stream
    flags = torch.zeros(1, dtype=torch.int32, device="cuda")
    wd = [torch.from_numpy(w0).cuda(), torch.empty(n, device="cuda")]
    md, vd = [moment(), moment()], [moment(), moment()]
    wh = torch.from_numpy(w0.copy()).pin_memory()
    wh_out = torch.empty(n, dtype=torch.float32).pin_memory()
    mh, vh = [moment(), moment()], [moment(), moment()]
    for t in range(1, 4):
        g = (r.standard_normal(n) * 1e-3).astype(np.float32)
        gh = torch.from_numpy(g).pin_memory()
        gd = gh.cuda()
        a, b = (t - 1) % 2, t % 2
        assert L.coat_adamw_dre_step(wd[a].data_ptr(), wd[b].data_ptr(), gd.data_ptr(), n, 128, cs(md[a]),
                                     cs(vd[a]), cs(md[b]), cs(vd[b]), C.byref(cfg), t, flags.data_ptr(), st) == 0
        assert L.coat_adamw_dre_step_host(wh.data_ptr(), wh_out.data_ptr(), gh.data_ptr(), n, 128, cs(mh[a]),
                                          cs(vh[a]), cs(mh[b]), cs(vh[b]), C.byref(cfg), t, flags.data_ptr(),
                                          chunk, st) == 0, L.coat_last_error()
        torch.cuda.synchronize()
        assert int(flags.item()) == 0
        assert torch.equal(wh_out, wd[b].cpu()), t
        for x, y in ((mh[b], md[b]), (vh[b], vd[b])):
            for key in ("codes", "scales", "k", "c"):
                assert torch.equal(x[key], y[key]), (t, key)
        wh.copy_(wh_out)
