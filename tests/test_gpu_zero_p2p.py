"""GPU: the ZeRO step with peer-memory collectives (coat_zero_step_p2p,
SURVEY.md 8(f)#3): reduce-scatter by direct loads from every rank's gradient
buffer, the fused step on the shard, all-gather by direct stores into every
rank's next-weight buffer, pipelined chunk by chunk.

One GPU is available, so N ranks are N "virtual ranks" on the same device:
each owns its own full gradient, current-weight and next-weight buffers and
its shard's optimizer state, and the peer pointer arrays point at the other
virtual ranks' buffers -- the same kernels and pipeline a multi-GPU node runs,
with NVLink replaced by local HBM.  Parity: the reduced gradient is the
rank-order fp32 sum (bf16 wire: of the exactly widened values), and the
gathered weights and every shard's state equal the checker's step of the whole
tensor on that sum (groups are independent, so sharded == whole,
SPEC.md:396), against both the C restatement and the reference itself.
The NVLink-SHARP (multimem) branch needs a multicast object, which a one-GPU
box cannot create (tools/mc_probe.py); it shares this pipeline and differs
only in the two copy kernels.
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


def _ptrs(ts):
    return (C.c_void_p * len(ts))(*[t.data_ptr() for t in ts])


def _bf16_round(x):
    b = x.view(np.uint32).astype(np.uint64)
    b = (b + 0x7FFF + ((b >> 16) & 1)) >> 16
    return (b.astype(np.uint32) << 16).view(np.float32)


@pytest.mark.parametrize("nranks,wire", [(1, "fp32"), (2, "fp32"), (4, "fp32"), (3, "bf16"), (8, "bf16")])
def test_p2p_step_virtual_ranks(checker, nranks, wire):
    import torch
    from paper_2410_19313_b200 import _lib
    L = _lib.lib
    n = 128 * 2100 + 128 * 7            # per-rank shard: ragged against the 2048-parameter round
    N = n * nranks
    r = rng(100 + nranks)
    w0 = (r.standard_normal(N) * 0.02).astype(np.float32)
    cfg = _lib.AdamWConfigC(**CFG)
    st = torch.cuda.current_stream().cuda_stream
    w_cur = [torch.from_numpy(w0).cuda() for _ in range(nranks)]
    w_next = [torch.full((N,), float("nan"), device="cuda") for _ in range(nranks)]
    m = [[_moment(n, torch), _moment(n, torch)] for _ in range(nranks)]
    v = [[_moment(n, torch), _moment(n, torch)] for _ in range(nranks)]
    g_shard = [torch.empty(n, device="cuda") for _ in range(nranks)]
    flags = [torch.zeros(1, dtype=torch.int32, device="cuda") for _ in range(nranks)]
    w_ref = w0.copy()
    mr, vr = checker.make_slot(N)
    for t in range(1, 4):
        gh = [(r.standard_normal(N) * 1e-3).astype(np.float32) for _ in range(nranks)]
        if wire == "bf16":
            gh = [_bf16_round(x) for x in gh]
            g = [torch.from_numpy(x).cuda().to(torch.bfloat16) for x in gh]
        else:
            g = [torch.from_numpy(x).cuda() for x in gh]
        gsum = gh[0].copy()
        for x in gh[1:]:
            gsum = (gsum + x).astype(np.float32)    # rank order, fp32 RN
        a, b = (t - 1) % 2, t % 2
        for rk in range(nranks):
            flags[rk].zero_()
            assert L.coat_zero_step_p2p(_ptrs(g), None, 0 if wire == "fp32" else 1, _ptrs(w_next), None,
                                        w_cur[rk].data_ptr(), w_next[rk].data_ptr(), N, 128,
                                        _cs(_lib, m[rk][a]), _cs(_lib, v[rk][a]), _cs(_lib, m[rk][b]),
                                        _cs(_lib, v[rk][b]), C.byref(cfg), t, g_shard[rk].data_ptr(),
                                        flags[rk].data_ptr(), rk, nranks, 2048 * 5, st) == 0, L.coat_last_error()
        torch.cuda.synchronize()
        assert all(int(f.item()) == 0 for f in flags)
        assert checker.step(w_ref, gsum, mr, vr, t - 1, CFG) == 0
        for rk in range(nranks):
            assert np.array_equal(g_shard[rk].cpu().numpy().view(np.uint32),
                                  gsum[rk * n:(rk + 1) * n].view(np.uint32)), (t, rk, "reduced gradient")
            assert np.array_equal(w_next[rk].cpu().numpy().view(np.uint32), w_ref.view(np.uint32)), (t, rk)
            sl = slice(rk * n, (rk + 1) * n)
            gs = slice(rk * n // 128, (rk + 1) * n // 128)
            for mine, full in ((m[rk][b], mr), (v[rk][b], vr)):
                assert np.array_equal(mine["codes"].cpu().numpy(), full["codes"][sl]), (t, rk)
                assert np.array_equal(mine["scales"].cpu().numpy().view(np.uint16).astype(np.uint32) << 16,
                                      full["scales"][gs].view(np.uint32)), (t, rk)
                assert np.array_equal(mine["k"].cpu().numpy(), full["k"][gs])
                assert np.array_equal(mine["c"].cpu().numpy(), full["c"][gs])
        w_cur, w_next = w_next, w_cur            # commit: the next weights become current


def test_p2p_step_nonfinite_gradient_leaves_current_weights(coat):
    """A NaN in one rank's gradient reaches the shard owner's reduced sum: its
    error word reports NonFiniteGradient (optimizer.cpp:104) and, the weights
    being double-buffered, every rank's current weights are untouched -- the
    caller keeps them by the OR of the error words."""
    import torch
    from paper_2410_19313_b200 import _lib
    L = _lib.lib
    nranks, n = 2, 128 * 1024
    N = n * nranks
    r = rng(7)
    w0 = torch.from_numpy((r.standard_normal(N) * 0.02).astype(np.float32)).cuda()
    w_cur = [w0.clone() for _ in range(nranks)]
    w_next = [torch.empty(N, device="cuda") for _ in range(nranks)]
    g = [torch.from_numpy((r.standard_normal(N) * 1e-3).astype(np.float32)).cuda() for _ in range(nranks)]
    g[0][n + 77] = float("nan")                  # rank 0's gradient, inside rank 1's shard
    cfg = _lib.AdamWConfigC(**CFG)
    st = torch.cuda.current_stream().cuda_stream
    fl = []
    for rk in range(nranks):
        m, v = [_moment(n, torch), _moment(n, torch)], [_moment(n, torch), _moment(n, torch)]
        f = torch.zeros(1, dtype=torch.int32, device="cuda")
        gs = torch.empty(n, device="cuda")
        assert L.coat_zero_step_p2p(_ptrs(g), None, 0, _ptrs(w_next), None, w_cur[rk].data_ptr(),
                                    w_next[rk].data_ptr(), N, 128, _cs(_lib, m[0]), _cs(_lib, v[0]),
                                    _cs(_lib, m[1]), _cs(_lib, v[1]), C.byref(cfg), 1, gs.data_ptr(), f.data_ptr(),
                                    rk, nranks, 0, st) == 0
        fl.append(f)
    torch.cuda.synchronize()
    word = int(fl[0].item()) | int(fl[1].item())
    assert int(fl[1].item()) & _lib.FLAG_NONFINITE_GRAD and not int(fl[0].item()) & _lib.FLAG_NONFINITE_GRAD
    assert L.coat_flags_to_status(word) == 4     # NonFiniteGradient for every rank after the OR
    assert all(torch.equal(w, w0) for w in w_cur)


def test_p2p_step_validates_before_any_work():
    from paper_2410_19313_b200 import _lib
    L = _lib.lib
    cfg = _lib.AdamWConfigC(**CFG)
    ms = _lib.MomentState(None, None, None, None)
    one = (C.c_void_p * 1)(16)
    # n_total not a multiple of 128 * nranks -> GeometryMismatch
    assert L.coat_zero_step_p2p(one, None, 0, one, None, 16, 16, 1000, 128, ms, ms, ms, ms, C.byref(cfg), 1, 16,
                                16, 0, 1, 0, None) == 2
    # bad rank, 17 ranks, multimem with bf16
    assert L.coat_zero_step_p2p(one, None, 0, one, None, 16, 16, 1024, 128, ms, ms, ms, ms, C.byref(cfg), 1, 16,
                                16, 1, 1, 0, None) == 5
    assert L.coat_zero_step_p2p(one, None, 0, one, None, 16, 16, 1024 * 17, 128, ms, ms, ms, ms, C.byref(cfg), 1,
                                16, 16, 0, 17, 0, None) == 5
    assert L.coat_zero_step_p2p(None, 16, 1, one, None, 16, 16, 1024, 128, ms, ms, ms, ms, C.byref(cfg), 1, 16,
                                16, 0, 1, 0, None) == 5


SHAPES = [(300,), (5, 128), (1000,), (64, 96), (7000,)]


def _peer_worker(port, grad_dtype, q):
    import os
    import sys
    from conftest import ROOT
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        from paper_2410_19313_b200 import coatsim
        from paper_2410_19313_b200.zero import PeerZeroAdamW
        dt = torch.bfloat16 if grad_dtype == "bf16" else torch.float32
        z = PeerZeroAdamW(SHAPES, coatsim.AdamWConfig(**CFG), grad_dtype=dt, chunk=2048 * 3)
        lay = z.layout
        r = np.random.default_rng(5)
        ws0 = [(r.standard_normal(int(np.prod(s))) * 0.02).astype(np.float32) for s in SHAPES]
        z.weights.copy_(lay.flatten([torch.from_numpy(w).reshape(s).cuda() for w, s in zip(ws0, SHAPES)]))
        grads = []
        for t in range(3):
            gs = [(r.standard_normal(int(np.prod(s))) * 1e-3).astype(np.float32) for s in SHAPES]
            gflat = lay.flatten([torch.from_numpy(g).reshape(s).cuda() for g, s in zip(gs, SHAPES)])
            z.grad.copy_(gflat.to(dt))
            grads.append([x.cpu().numpy() for x in lay.views(z.grad.float())])
            z.step()
        torch.cuda.synchronize()
        w = [x.cpu().numpy().copy() for x in lay.views(z.weights)]
        z.grad[lay.offsets[2] + 5] = float("nan")
        before = z.weights.clone()
        raised = None
        try:
            z.step()
        except coatsim.Error as e:
            raised = type(e).__name__
        q.put(("ok", {"w0": ws0, "grads": grads, "w": w, "raised": raised, "same": bool(torch.equal(z.weights, before)),
                      "steps": z.step_count, "mc": z.uses_multicast}))
    except Exception:
        import traceback
        q.put(("err", traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("grad_dtype", ["fp32", "bf16"])
def test_peer_zero_adamw_symmetric_memory(checker, grad_dtype):
    """zero.PeerZeroAdamW end to end on torch symmetric memory (one rank: the
    one GPU), per-tensor parity against the checker, and the reference's
    NonFiniteGradient commit semantics on the double-buffered weights."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_peer_worker, args=(port, grad_dtype, q))
    p.start()
    status, res = q.get(timeout=600)
    p.join(timeout=120)
    assert status == "ok", res
    for i, s in enumerate(SHAPES):
        n = int(np.prod(s))
        w = res["w0"][i].copy()
        m, v = checker.make_slot(n)
        for t in range(3):
            assert checker.step(w, res["grads"][t][i].reshape(-1), m, v, t, CFG) == 0
        assert np.array_equal(res["w"][i].reshape(-1).view(np.uint32), w.view(np.uint32)), (grad_dtype, i)
    assert res["raised"] == "NonFiniteGradient" and res["same"] and res["steps"] == 3, res


def _ipc_worker(rank, ws, q_out, q_peers, barrier):
    import ctypes as C
    import sys
    from conftest import ROOT
    sys.path.insert(0, ROOT)
    import torch
    torch.cuda.set_device(0)
    try:
        from paper_2410_19313_b200 import _lib
        L = _lib.lib
        n = 128 * 1500 + 128 * 3
        N = n * ws
        r = np.random.default_rng(77)
        w0 = (r.standard_normal(N) * 0.02).astype(np.float32)
        g = torch.empty(N, device="cuda")
        w = [torch.from_numpy(w0).cuda(), torch.full((N,), float("nan"), device="cuda")]
        # every process maps every other process's gradient and weight buffers (CUDA IPC)
        for k in range(ws):
            if k != rank:
                q_peers[k].put((rank, g, w[0], w[1]))
        peers = {rank: (g, w[0], w[1])}
        while len(peers) < ws:
            rk, a, b, c = q_peers[rank].get(timeout=300)
            peers[rk] = (a, b, c)
        barrier.wait()
        gp = (C.c_void_p * ws)(*[peers[k][0].data_ptr() for k in range(ws)])
        wp = [(C.c_void_p * ws)(*[peers[k][1 + j].data_ptr() for k in range(ws)]) for j in range(2)]
        m, v = [_moment(n, torch), _moment(n, torch)], [_moment(n, torch), _moment(n, torch)]
        flags = torch.zeros(1, dtype=torch.int32, device="cuda")
        g_shard = torch.empty(n, device="cuda")
        cfg = _lib.AdamWConfigC(**CFG)
        st = torch.cuda.current_stream().cuda_stream
        grads = []
        cur = 0
        for t in range(1, 4):
            gh = (np.random.default_rng(1000 * t + rank).standard_normal(N) * 1e-3).astype(np.float32)
            grads.append(gh)
            g.copy_(torch.from_numpy(gh))
            torch.cuda.synchronize()
            barrier.wait()                      # every rank's gradients are in place
            a, b = (t - 1) % 2, t % 2
            assert L.coat_zero_step_p2p(gp, None, 0, wp[1 - cur], None, w[cur].data_ptr(), w[1 - cur].data_ptr(),
                                        N, 128, _cs(_lib, m[a]), _cs(_lib, v[a]), _cs(_lib, m[b]), _cs(_lib, v[b]),
                                        C.byref(cfg), t, g_shard.data_ptr(), flags.data_ptr(), rank, ws, 2048 * 7,
                                        st) == 0, L.coat_last_error()
            torch.cuda.synchronize()
            assert int(flags.item()) == 0
            barrier.wait()                      # every rank's stores into every next-weight buffer landed
            cur = 1 - cur
        st_out = {k: m[1][k].cpu().numpy().copy() for k in ("codes", "k", "c")}
        st_out["scales"] = m[1]["scales"].cpu().numpy().copy()
        q_out.put((rank, "ok", {"w": w[cur].cpu().numpy().copy(), "grads": grads, "w0": w0, "m": st_out, "n": n}))
        barrier.wait()                          # peers keep their buffers alive until everyone is done
    except Exception:
        import traceback
        q_out.put((rank, "err", traceback.format_exc()))


@pytest.mark.parametrize("ws", [2, 3])
def test_p2p_step_separate_processes_ipc(checker, ws):
    """coat_zero_step_p2p across real process boundaries: every rank is its own
    process on the one GPU and maps the other ranks' gradient and weight
    buffers through CUDA IPC (torch.multiprocessing), as ranks on an NVLink
    node map each other's memory.  Final weights on every rank and rank 0's
    first-moment shard against the checker's step on the rank-order sum."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q_out, barrier = ctx.Queue(), ctx.Barrier(ws)
    q_peers = [ctx.Queue() for _ in range(ws)]
    procs = [ctx.Process(target=_ipc_worker, args=(r, ws, q_out, q_peers, barrier)) for r in range(ws)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(ws):
        rk, status, d = q_out.get(timeout=600)
        assert status == "ok", f"rank {rk}: {d}"
        res[rk] = d
    for p in procs:
        p.join(timeout=120)
    n = res[0]["n"]
    N = n * ws
    w_ref = res[0]["w0"].copy()
    m, v = checker.make_slot(N)
    for t in range(3):
        gsum = res[0]["grads"][t].copy()
        for rk in range(1, ws):
            gsum = (gsum + res[rk]["grads"][t]).astype(np.float32)
        assert checker.step(w_ref, gsum, m, v, t, CFG) == 0
    for rk in range(ws):
        assert np.array_equal(res[rk]["w"].view(np.uint32), w_ref.view(np.uint32)), rk
    mine = res[0]["m"]
    assert np.array_equal(mine["codes"], m["codes"][:n])
    assert np.array_equal(mine["k"], m["k"][:n // 128]) and np.array_equal(mine["c"], m["c"][:n // 128])


@pytest.mark.parametrize("env", [{"COAT_P2P_FUSED_AG": "0"}, {"COAT_K1_EW": "7"}],
                         ids=["separate-broadcast", "ew7-fallback"])
def test_p2p_step_separate_broadcast_path(env):
    """COAT_P2P_FUSED_AG=0: the all-gather by the separate P2P broadcast kernel
    instead of K1's own peer stores; COAT_K1_EW=7: the fused variant exists
    for the default layout only, so the step falls back to the broadcast --
    the virtual-rank parity cases pass on both (the default runs them with the
    all-gather fused into K1)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                          "tests/test_gpu_zero_p2p.py", "-k", "virtual_ranks"],
                         cwd=root, env=dict(os.environ, **env), capture_output=True, text=True, timeout=900)
    tail = (out.stdout + out.stderr)[-3000:]
    assert out.returncode == 0, tail
    assert " passed" in out.stdout and " failed" not in out.stdout, tail
