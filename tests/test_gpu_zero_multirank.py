"""GPU, world size 2 and 4: the ZeRO-sharded step THROUGH THE FUSED KERNEL.

Every rank is a separate process on the one available GPU (gloo for the
collectives, staged through host memory; NCCL refuses two ranks on one
device).  Each rank runs ZeroAdamW.step -- reduce-scatter -> K1 on its
128-aligned shard -> error-word agreement -> all-gather -- for 3 steps over a
multi-tensor FlatLayout, every rank with its own gradients.  The test then
checks, bit for bit:
  * the gathered weights on every rank, and every rank's E4M3 codes, BF16
    scales, k and c of its shard, against BOTH CPU checkers -- the C port and
    the unmodified reference (oracle/_ref) -- stepping each tensor alone on the
    summed gradients (optimizer.cpp:101-114; shard independence);
  * a non-finite gradient injected on ONE rank, inside ANOTHER rank's shard:
    every rank raises NonFiniteGradient and nothing changes anywhere
    (optimizer.cpp:104) -- the cross-rank error agreement on the kernel.
Gradients are multiples of 2^-26 with |k| <= 2^22 (outliers included), so
their sum over <= 4 ranks is exact in fp32 and the summation order of the
collective cannot matter.
"""
import os
import socket

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

CFG = {"beta1": 0.9, "beta2": 0.999, "lr": 1e-3, "weight_decay": 0.1, "eps": 1e-8}
SHAPES = [(300,), (5, 128), (1000,), (3, 7, 11), (64, 96), (7000,)]
STEPS = 3


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _weights(i, n):
    r = np.random.default_rng(1000 + i)
    return (r.standard_normal(n) * 0.02).astype(np.float32)


def _grad(t, i, rank, n):
    """Exact-sum gradients: k * 2^-26, |k| <= 2^16, 1% outliers x 64."""
    r = np.random.default_rng(50_000 + 1000 * t + 10 * i + rank)
    k = r.integers(-(1 << 16), 1 << 16, n).astype(np.float64)
    k[r.random(n) < 0.01] *= 64
    return (k * 2.0 ** -26).astype(np.float32)


def _worker(rank, ws, port, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        from paper_2410_19313_b200 import coatsim
        from paper_2410_19313_b200.zero import ZeroAdamW
        z = ZeroAdamW(SHAPES, coatsim.AdamWConfig(**CFG), device="cuda")
        lay = z.layout
        w = lay.flatten([torch.from_numpy(_weights(i, int(np.prod(s)))).reshape(s).cuda()
                         for i, s in enumerate(SHAPES)])
        for t in range(STEPS):
            g = lay.flatten([torch.from_numpy(_grad(t, i, rank, int(np.prod(s)))).reshape(s).cuda()
                             for i, s in enumerate(SHAPES)])
            z.step(w, g)
        torch.cuda.synchronize()

        def state():
            out = {}
            for name, st in (("m", z.slot.m), ("v", z.slot.v)):
                out[name + "codes"] = st.quantized.codes.cpu().numpy().copy()
                out[name + "scales"] = st.quantized.scales.float().cpu().numpy().copy()
                out[name + "k"] = st.k.cpu().numpy().copy()
                out[name + "c"] = st.c.cpu().numpy().copy()
            return out

        res = {"w": w.cpu().numpy().copy(), "state": state(), "lo": z.lo, "hi": z.hi, "steps": z.step_count}
        # NaN on rank 1 only, at an index owned by rank 0's shard
        g = lay.flatten([torch.from_numpy(_grad(STEPS, i, rank, int(np.prod(s)))).reshape(s).cuda()
                         for i, s in enumerate(SHAPES)])
        if rank == 1:
            g[lay.offsets[1] + 3] = float("nan")
        w_before = w.clone()
        raised = None
        try:
            z.step(w, g)
        except coatsim.Error as e:
            raised = type(e).__name__
        torch.cuda.synchronize()
        after = state()
        res["nan"] = {"raised": raised, "w_same": bool(torch.equal(w, w_before)), "steps": z.step_count,
                      "state_same": all(np.array_equal(after[k], res["state"][k]) for k in after)}
        q.put((rank, "ok", res))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, "err", traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def _reference(oracle, lay, ws):
    """Per-tensor step on the summed gradients (the single-process step)."""
    out = []
    for i, s in enumerate(SHAPES):
        n = int(np.prod(s))
        w = _weights(i, n)
        m, v = oracle.make_slot(n)
        for t in range(STEPS):
            g = np.zeros(n, np.float32)
            for r in range(ws):
                g = g + _grad(t, i, r, n)
            assert oracle.step(w, g, m, v, t, CFG) == 0
        out.append((w, m, v))
    return out


@pytest.mark.parametrize("ws", [2, 4])
def test_zero_multirank_kernel_matches_reference(ws, port, ref):
    import torch.multiprocessing as mp
    from paper_2410_19313_b200.zero import FlatLayout
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, ws, p, q)) for r in range(ws)]
    for pr in procs:
        pr.start()
    results = {}
    for _ in range(ws):
        rank, status, res = q.get(timeout=600)
        assert status == "ok", f"rank {rank}: {res}"
        results[rank] = res
    for pr in procs:
        pr.join(timeout=120)
    assert all(pr.exitcode == 0 for pr in procs)

    lay = FlatLayout.build(SHAPES, ws)
    for checker in (port, ref):
        expect = _reference(checker, lay, ws)
        for rank, res in results.items():
            assert res["steps"] == STEPS
            lo, hi = res["lo"], res["hi"]
            for i, (w, m, v) in enumerate(expect):
                off, n = lay.offsets[i], lay.numels[i]
                assert np.array_equal(res["w"][off:off + n].view(np.uint32), w.view(np.uint32)), \
                    f"{checker.kind} rank {rank} tensor {i} weights"
                npad = -(-n // 128) * 128
                # the part of tensor i inside this rank's shard
                a, b = max(off, lo), min(off + npad, hi)
                if a >= b:
                    continue
                for name, st in (("m", m), ("v", v)):
                    got = res["state"][name + "codes"][a - lo:b - lo]
                    assert np.array_equal(got, st["codes"][a - off:b - off]), \
                        f"{checker.kind} rank {rank} tensor {i} {name} codes"
                    ga, gb = (a - lo) // 128, (b - lo) // 128
                    ra, rb = (a - off) // 128, (b - off) // 128
                    for key in ("scales", "k", "c"):
                        assert np.array_equal(res["state"][name + key][ga:gb].view(np.uint32),
                                              np.ascontiguousarray(st[key][ra:rb]).view(np.uint32)), \
                            f"{checker.kind} rank {rank} tensor {i} {name} {key}"
    # cross-rank error agreement on the kernel path
    for rank, res in results.items():
        nan = res["nan"]
        assert nan["raised"] == "NonFiniteGradient", (rank, nan)
        assert nan["w_same"] and nan["state_same"] and nan["steps"] == STEPS, (rank, nan)
