"""ZeRO sharding of the FP8-DRE AdamW step (paper_2410_19313_b200/zero.py).

CPU (gloo, world_size 2): the flat 128-aligned layout, the reduce-scatter /
all-gather plumbing and the shard-independence property the sharded step
relies on -- each rank steps only its shard (here with the oracle, as the
checker) and the gathered result must equal, bit for bit, the reference's
per-tensor step on the summed gradients (optimizer.cpp:101-114).
GPU (world_size 1, NCCL): ZeroAdamW.step through the fused kernel equals
coatsim.step on the same buffers, including the error semantics.
"""
import os
import socket

import numpy as np
import pytest

from conftest import ROOT

CFG = {"beta1": 0.9, "beta2": 0.999, "lr": 1e-3, "weight_decay": 0.1, "eps": 1e-8}
SHAPES = [(300,), (5, 128), (1000,), (3, 7, 11)]


def _layout():
    from paper_2410_19313_b200.zero import FlatLayout
    return FlatLayout


def test_flat_layout_alignment_and_round_trip():
    import torch
    FlatLayout = _layout()
    for ws in (1, 2, 3, 8):
        lay = FlatLayout.build(SHAPES, ws)
        assert all(o % 128 == 0 for o in lay.offsets)
        assert lay.total % (128 * ws) == 0 and lay.shard_numel % 128 == 0
        assert lay.offsets[-1] + lay.numels[-1] <= lay.total
        shards = [lay.shard(r) for r in range(ws)]
        assert shards[0][0] == 0 and shards[-1][1] == lay.total
        assert all(a[1] == b[0] for a, b in zip(shards, shards[1:]))
    lay = FlatLayout.build(SHAPES, 2)
    ts = [torch.randn(s) for s in SHAPES]
    flat = lay.flatten(ts)
    for a, b in zip(ts, lay.views(flat)):
        assert torch.equal(a, b)
    # padding is zero (pad_flat, optimizer.cpp:24-38)
    mask = torch.ones(lay.total, dtype=torch.bool)
    for o, n in zip(lay.offsets, lay.numels):
        mask[o:o + n] = False
    assert torch.all(flat[mask] == 0)


def test_flat_layout_errors():
    from paper_2410_19313_b200 import coatsim
    FlatLayout = _layout()
    with pytest.raises(coatsim.InvalidSpec):
        FlatLayout.build([(0, 4)], 2)
    with pytest.raises(coatsim.InvalidSpec):
        FlatLayout.build([(4,)], 0)
    lay = FlatLayout.build([(4,)], 1)
    import torch
    with pytest.raises(coatsim.ShapeMismatch):
        lay.flatten([torch.zeros(5)])


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _zero_worker(rank, ws, port, steps, q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import torch
    import torch.distributed as dist
    from pyoracle import Oracle
    from paper_2410_19313_b200.zero import FlatLayout, all_gather_params, reduce_scatter_grads

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        o = Oracle("port")
        lay = FlatLayout.build(SHAPES, ws)
        lo, hi = lay.shard(rank)
        w_t = [o.generate(0, (int(np.prod(s)),), 0.0, 100.0, 1 + i) * np.float32(0.02) for i, s in enumerate(SHAPES)]
        w_full = lay.flatten([torch.from_numpy(a).reshape(s) for a, s in zip(w_t, SHAPES)])
        m, v = o.make_slot(hi - lo)          # this rank's shard of the state
        g_shard = torch.empty(hi - lo)
        for t in range(steps):
            g_t = [o.generate(0, (int(np.prod(s)),), 0.01, 100.0, 100 + 10 * t + 3 * i + rank) * np.float32(1e-3)
                   for i, s in enumerate(SHAPES)]
            g_full = lay.flatten([torch.from_numpy(a).reshape(s) for a, s in zip(g_t, SHAPES)])
            reduce_scatter_grads(g_full, g_shard)
            w_np = w_full.numpy()
            shard = np.ascontiguousarray(w_np[lo:hi])
            assert o.step(shard, g_shard.numpy(), m, v, t, CFG) == 0
            w_full[lo:hi] = torch.from_numpy(shard)
            all_gather_params(w_full, w_full[lo:hi].clone())
        # gather every rank's state shard (test-side) for the comparison
        state = {}
        for name, st in (("m", m), ("v", v)):
            for key in ("codes", "scales", "k", "c"):
                a = torch.from_numpy(np.ascontiguousarray(st[key]).view(np.uint8 if key == "codes" else np.uint32)
                                     .astype(np.int64))
                out = torch.empty(a.numel() * ws, dtype=torch.int64)
                dist.all_gather_into_tensor(out, a)
                state[name + key] = out.numpy()
        if rank == 0:
            q.put(("ok", w_full.numpy().copy(), state))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put(("err", repr(e), None))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("ws", [2])
def test_zero_sharded_step_gloo_matches_reference(ws, port):
    import torch.multiprocessing as mp
    steps = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = _free_port()
    procs = [ctx.Process(target=_zero_worker, args=(r, ws, p, steps, q)) for r in range(ws)]
    for pr in procs:
        pr.start()
    status, w_flat, state = q.get(timeout=300)
    for pr in procs:
        pr.join(timeout=120)
    assert status == "ok", w_flat
    assert all(pr.exitcode == 0 for pr in procs)
    # the reference: per-tensor step on the summed gradients (sum of 2 floats is order-free)
    FlatLayout = _layout()
    lay = FlatLayout.build(SHAPES, ws)
    for i, s in enumerate(SHAPES):
        n = int(np.prod(s))
        w = port.generate(0, (n,), 0.0, 100.0, 1 + i) * np.float32(0.02)
        m, v = port.make_slot(n)
        for t in range(steps):
            g = np.zeros(n, np.float32)
            for r in range(ws):
                g = g + port.generate(0, (n,), 0.01, 100.0, 100 + 10 * t + 3 * i + r) * np.float32(1e-3)
            assert port.step(w, g, m, v, t, CFG) == 0
        off = lay.offsets[i]
        assert np.array_equal(w_flat[off:off + n].view(np.uint32), w.view(np.uint32)), f"tensor {i} weights"
        npad = -(-n // 128) * 128
        for name, st in (("m", m), ("v", v)):
            got = state[name + "codes"][off:off + npad].astype(np.uint8)
            assert np.array_equal(got, st["codes"]), f"tensor {i} {name} codes"
            g0 = off // 128
            for key in ("scales", "k", "c"):
                got = state[name + key][g0:g0 + npad // 128].astype(np.uint32)
                assert np.array_equal(got, np.ascontiguousarray(st[key]).view(np.uint32)), f"tensor {i} {name} {key}"


@pytest.mark.gpu
def test_zero_step_nccl_world1_equals_step():
    import torch
    import torch.distributed as dist
    from paper_2410_19313_b200 import coatsim
    from paper_2410_19313_b200.zero import ZeroAdamW
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        cfg = coatsim.AdamWConfig(**CFG)
        z = ZeroAdamW(SHAPES, cfg)
        lay = z.layout
        gen = torch.Generator(device="cuda").manual_seed(5)
        w = lay.flatten([torch.randn(s, device="cuda", generator=gen) * 0.02 for s in SHAPES])
        w_ref = w.clone()
        slot = coatsim.make_slot([lay.total])
        for _ in range(3):
            g = lay.flatten([torch.randn(s, device="cuda", generator=gen) * 1e-3 for s in SHAPES])
            z.step(w, g)
            coatsim.step(w_ref, g, slot, cfg)
        assert torch.equal(w.view(torch.int32), w_ref.view(torch.int32))
        assert torch.equal(z.slot.m.quantized.codes, slot.m.quantized.codes)
        assert torch.equal(z.slot.v.quantized.codes, slot.v.quantized.codes)
        # NonFiniteGradient: nothing changes
        g = torch.zeros(lay.total, device="cuda")
        g[7] = float("nan")
        before = w.clone()
        with pytest.raises(coatsim.NonFiniteGradient):
            z.step(w, g)
        assert torch.equal(w, before) and z.step_count == 3
    finally:
        dist.destroy_process_group()
