"""GPU: the C-ABI ZeRO step (coat_zero_step) over a real
NCCL communicator built with the library's own helpers.

Only one GPU is available to the tests, so the communicator has one rank:
the reduce-scatter, error-word all-reduce and all-gather run through NCCL
with their degenerate (identity) semantics, and the result must equal the
single-GPU coat_adamw_dre_step bit for bit (optimizer.cpp:101-114); with a
non-finite gradient nothing may change (optimizer.cpp:104).  The N > 1 host
logic is covered by tests/test_zero.py (gloo, 2 ranks).
"""
import ctypes as C

import numpy as np
import pytest

from conftest import rng

pytestmark = pytest.mark.gpu

CFG = {"beta1": 0.9, "beta2": 0.999, "lr": 1e-3, "weight_decay": 0.1, "eps": 1e-8}


def _moment(n, torch):
    ng = n // 128
    return {"codes": torch.zeros(n, dtype=torch.uint8, device="cuda"),
            "scales": torch.full((ng,), 0x3B00, dtype=torch.int16, device="cuda"),   # 2^-9 (make_slot)
            "k": torch.ones(ng, device="cuda"), "c": torch.ones(ng, device="cuda")}


def _cs(_lib, mm):
    return _lib.MomentState(mm["codes"].data_ptr(), mm["scales"].data_ptr(), mm["k"].data_ptr(), mm["c"].data_ptr())


@pytest.fixture(scope="module")
def comm():
    from paper_2410_19313_b200 import _lib
    L = _lib.lib
    uid = (C.c_uint8 * 128)()
    assert L.coat_nccl_unique_id(uid) == 0, L.coat_last_error()
    c = C.c_void_p()
    assert L.coat_nccl_comm_init(C.byref(c), 1, uid, 0) == 0, L.coat_last_error()
    yield c
    assert L.coat_nccl_comm_destroy(c) == 0


def test_zero_step_one_rank_equals_single_gpu_step(comm):
    import torch
    from paper_2410_19313_b200 import _lib
    L = _lib.lib
    n = 128 * 25000
    r = rng(41)
    w0 = (r.standard_normal(n) * 0.02).astype(np.float32)
    cfg = _lib.AdamWConfigC(**CFG)
    st = torch.cuda.current_stream().cuda_stream
    flags = torch.zeros(1, dtype=torch.int32, device="cuda")
    # single-GPU ping-pong
    wp = [torch.from_numpy(w0).cuda(), torch.empty(n, device="cuda")]
    mp, vp = [_moment(n, torch), _moment(n, torch)], [_moment(n, torch), _moment(n, torch)]
    # ZeRO step
    wz = torch.from_numpy(w0).cuda()
    mz, vz = [_moment(n, torch), _moment(n, torch)], [_moment(n, torch), _moment(n, torch)]
    g_shard = torch.empty(n, device="cuda")
    w_scr = torch.empty(n, device="cuda")
    for t in range(1, 5):
        g = torch.from_numpy((r.standard_normal(n) * 1e-3).astype(np.float32)).cuda()
        a, b = (t - 1) % 2, t % 2
        flags.zero_()
        assert L.coat_adamw_dre_step(wp[a].data_ptr(), wp[b].data_ptr(), g.data_ptr(), n, 128, _cs(_lib, mp[a]),
                                     _cs(_lib, vp[a]), _cs(_lib, mp[b]), _cs(_lib, vp[b]), C.byref(cfg), t,
                                     flags.data_ptr(), st) == 0
        torch.cuda.synchronize()
        assert int(flags.item()) == 0
        assert L.coat_zero_step(wz.data_ptr(), g.data_ptr(), n, 128, _cs(_lib, mz[a]), _cs(_lib, vz[a]),
                                _cs(_lib, mz[b]), _cs(_lib, vz[b]), C.byref(cfg), t, g_shard.data_ptr(),
                                w_scr.data_ptr(), flags.data_ptr(), comm, 0, 1, st) == 0, L.coat_last_error()
        torch.cuda.synchronize()
        assert int(flags.item()) == 0
        assert torch.equal(wz, wp[b]), t
        for x, y in ((mz[b], mp[b]), (vz[b], vp[b])):
            for key in ("codes", "scales", "k", "c"):
                assert torch.equal(x[key], y[key]), (t, key)


def test_zero_step_nonfinite_gradient_changes_nothing(comm):
    import torch
    from paper_2410_19313_b200 import _lib
    L = _lib.lib
    n = 128 * 4096
    r = rng(43)
    w0 = torch.from_numpy((r.standard_normal(n) * 0.02).astype(np.float32)).cuda()
    w = w0.clone()
    g = torch.from_numpy((r.standard_normal(n) * 1e-3).astype(np.float32)).cuda()
    g[12345] = float("nan")
    m, v = [_moment(n, torch), _moment(n, torch)], [_moment(n, torch), _moment(n, torch)]
    flags = torch.zeros(1, dtype=torch.int32, device="cuda")
    cfg = _lib.AdamWConfigC(**CFG)
    g_shard, w_scr = torch.empty(n, device="cuda"), torch.empty(n, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    assert L.coat_zero_step(w.data_ptr(), g.data_ptr(), n, 128, _cs(_lib, m[0]), _cs(_lib, v[0]), _cs(_lib, m[1]),
                            _cs(_lib, v[1]), C.byref(cfg), 1, g_shard.data_ptr(), w_scr.data_ptr(),
                            flags.data_ptr(), comm, 0, 1, st) == 0
    torch.cuda.synchronize()
    fl = int(flags.item())
    assert fl & _lib.FLAG_NONFINITE_GRAD
    assert L.coat_flags_to_status(fl) == 4   # NonFiniteGradient
    assert torch.equal(w, w0)


def test_zero_step_validates_before_any_work(comm):
    from paper_2410_19313_b200 import _lib
    L = _lib.lib
    cfg = _lib.AdamWConfigC(**CFG)
    ms = _lib.MomentState(None, None, None, None)
    # n_total not a multiple of 128 * nranks -> GeometryMismatch, nothing launched
    assert L.coat_zero_step(1, 1, 1000, 128, ms, ms, ms, ms, C.byref(cfg), 1, 1, 1, 1, comm, 0, 1, None) == 2
    assert L.coat_zero_step(1, 1, 1024, 128, ms, ms, ms, ms, C.byref(cfg), 1, 1, 1, 1, comm, 1, 1, None) == 5
