"""ZeRO-sharded FP8-DRE AdamW over torch.distributed (one process per GPU).

The reference steps one tensor at a time (coatsim::step, optimizer.cpp:101-114)
and has no distributed code.  Its Dynamic Range Expansion statistics are per
1x128 group (expand.cpp:57-83), so a flat buffer whose tensors each start on a
128-element boundary can be cut into 128-aligned shards that are stepped
independently, bit for bit equal to the per-tensor reference step
("shard independence"; tests/test_zero.py checks
it with the oracle on 2 gloo ranks).

Per step, rank r:
  1. reduce-scatter of the full fp32 gradient buffer (sum) -> its shard,
  2. the fused K1 kernel (coatsim._step_launch) on its shard of the weights
     and its shard of the FP8-DRE state (the state is never communicated); the
     new weight shard goes to a scratch buffer,
  3. an all-reduce of the 5-bit error word, so every rank commits exactly
     what the single-process step would commit for the union of the shards
     (coatsim._step_commit: NonFiniteGradient anywhere -> nothing changes
     anywhere),
  4. when the weights change: all-gather of the scratch shards straight into
     the full weight buffer -- the all-gather IS the commit, so the sharded
     step moves no extra bytes (world size 1: one copy).

NCCL over NVLink on B200 (``backend="nccl"``); the same code runs on gloo for
the CPU tests of the plumbing.  Gradient averaging is the caller's choice
(``grad_op="sum"`` like the reference, which just consumes g).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import torch
import torch.distributed as dist

from . import _lib, coatsim

GROUP = coatsim.DRE_GROUP


def _round_up(x: int, m: int) -> int:
    return -(-x // m) * m


@dataclass(frozen=True)
class FlatLayout:
    """Tensors packed into one flat fp32 buffer, each padded to a multiple of
    128 elements (optimizer.cpp:24-38 pad_flat), the total padded to a
    multiple of 128 * world_size so every rank owns an equal 128-aligned shard."""

    shapes: tuple
    offsets: tuple
    numels: tuple
    total: int
    world_size: int

    @staticmethod
    def build(shapes: Sequence[Sequence[int]], world_size: int = 1) -> "FlatLayout":
        if world_size < 1:
            raise coatsim.InvalidSpec("world_size must be >= 1")
        offs, numels, cur = [], [], 0
        norm = []
        for s in shapes:
            s = tuple(int(d) for d in s)
            if any(d <= 0 for d in s):
                raise coatsim.InvalidSpec("tensor dimensions must be positive")
            n = 1
            for d in s:
                n *= d
            norm.append(s)
            offs.append(cur)
            numels.append(n)
            cur += _round_up(n, GROUP)
        total = _round_up(max(cur, 1), GROUP * world_size)
        return FlatLayout(tuple(norm), tuple(offs), tuple(numels), total, world_size)

    @property
    def shard_numel(self) -> int:
        return self.total // self.world_size

    def shard(self, rank: int) -> tuple[int, int]:
        lo = rank * self.shard_numel
        return lo, lo + self.shard_numel

    def flatten(self, tensors: Sequence[torch.Tensor], out: torch.Tensor | None = None) -> torch.Tensor:
        if len(tensors) != len(self.shapes):
            raise coatsim.ShapeMismatch("flatten: tensor count differs from the layout")
        dev = tensors[0].device if tensors else None
        if out is None:
            out = torch.zeros(self.total, dtype=torch.float32, device=dev)
        else:
            out.zero_()
        for t, s, o, n in zip(tensors, self.shapes, self.offsets, self.numels):
            if tuple(t.shape) != s:
                raise coatsim.ShapeMismatch("flatten: shape differs from the layout")
            out[o:o + n].copy_(t.reshape(-1))
        return out

    def views(self, flat: torch.Tensor) -> list[torch.Tensor]:
        return [flat[o:o + n].view(s) for s, o, n in zip(self.shapes, self.offsets, self.numels)]


def _world(group) -> tuple[int, int]:
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(group), dist.get_rank(group)
    return 1, 0


def _host_staged(t: torch.Tensor, group) -> bool:
    """gloo has no CUDA reduce-scatter / all-gather-into-tensor: stage CUDA
    buffers through host memory (functional multi-rank runs on one GPU --
    tests/test_gpu_zero_multirank.py; NCCL takes the device buffers as is)."""
    return t.is_cuda and dist.get_backend(group) == "gloo"


def reduce_scatter_grads(g_full: torch.Tensor, g_shard: torch.Tensor, group=None, grad_op: str = "sum") -> None:
    """g_shard = (sum over ranks of g_full)[this rank's shard]; grad_op="avg" divides by world size."""
    ws, _ = _world(group)
    if ws == 1:
        if g_shard.data_ptr() != g_full.data_ptr():
            g_shard.copy_(g_full[:g_shard.numel()])
    elif _host_staged(g_full, group):
        out = torch.empty(g_shard.shape, dtype=g_shard.dtype)
        dist.reduce_scatter_tensor(out, g_full.cpu(), op=dist.ReduceOp.SUM, group=group)
        g_shard.copy_(out)
    else:
        dist.reduce_scatter_tensor(g_shard, g_full, op=dist.ReduceOp.SUM, group=group)
    if grad_op == "avg" and ws > 1:
        g_shard.div_(ws)
    elif grad_op not in ("sum", "avg"):
        raise coatsim.InvalidSpec(f"grad_op must be 'sum' or 'avg', not {grad_op!r}")


def all_gather_params(w_full: torch.Tensor, w_shard: torch.Tensor, group=None) -> None:
    """Every rank's shard -> w_full on every rank (rank r's shard lands at
    [r * n_shard, (r + 1) * n_shard)).  w_shard may alias its slot in w_full."""
    ws, rank = _world(group)
    if ws > 1 and _host_staged(w_full, group):
        out = torch.empty(w_full.shape, dtype=w_full.dtype)
        dist.all_gather_into_tensor(out, w_shard.cpu(), group=group)
        w_full.copy_(out)
    elif ws > 1:
        dist.all_gather_into_tensor(w_full, w_shard, group=group)
    else:
        n = w_shard.numel()
        if w_shard.data_ptr() != w_full.data_ptr():
            w_full[:n].copy_(w_shard)


def _all_flags(flags: torch.Tensor, group) -> int:
    """OR of the device error words of all ranks (as 5 one-bit lanes, MAX-reduced)."""
    ws, _ = _world(group)
    if ws == 1:
        return int(flags.item())
    bits = torch.stack([(flags >> i) & 1 for i in range(5)]).reshape(-1).to(torch.int32)
    if _host_staged(bits, group):
        bits = bits.cpu()
    dist.all_reduce(bits, op=dist.ReduceOp.MAX, group=group)
    v = 0
    for i, b in enumerate(bits.tolist()):
        v |= (int(b) & 1) << i
    return v


class ZeroAdamW:
    """FP8-DRE AdamW with the optimizer state partitioned over the ranks of
    ``group`` (ZeRO stage 1/2): this rank owns parameters [lo, hi) of the flat
    layout and only their E4M3 + DRE state."""

    def __init__(self, shapes: Sequence[Sequence[int]], cfg: coatsim.AdamWConfig | None = None, group=None,
                 device=None, grad_op: str = "sum"):
        self.group = group
        self.world_size, self.rank = _world(group)
        self.layout = FlatLayout.build(shapes, self.world_size)
        self.lo, self.hi = self.layout.shard(self.rank)
        self.cfg = cfg or coatsim.AdamWConfig()
        self.grad_op = grad_op
        device = torch.device(device or "cuda")
        self.slot = coatsim.make_slot([self.hi - self.lo], device=device)
        self.g_shard = torch.empty(self.hi - self.lo, dtype=torch.float32, device=device)

    @property
    def step_count(self) -> int:
        return self.slot.step

    def step(self, w_full: torch.Tensor, g_full: torch.Tensor) -> None:
        """One optimizer step on flat buffers of ``layout.total`` fp32 elements.
        w_full is updated in place on every rank; raises the reference's
        exception (the same one on every rank) on non-finite values."""
        n = self.layout.total
        if w_full.numel() != n or g_full.numel() != n:
            raise coatsim.ShapeMismatch("ZeroAdamW.step: buffers do not match the flat layout")
        if not w_full.is_contiguous() or not g_full.is_contiguous():
            raise coatsim.InvalidSpec("ZeroAdamW.step: buffers must be contiguous")
        reduce_scatter_grads(g_full, self.g_shard, self.group, self.grad_op)
        coatsim._step_launch(w_full[self.lo:self.hi], self.g_shard, self.slot, self.cfg)
        flags = _all_flags(self.slot._flags.t, self.group)
        weights_change = not (flags & (_lib.FLAG_NONFINITE_GRAD | _lib.FLAG_CONTRACT))
        try:
            coatsim._step_commit(None, self.slot, flags)
        finally:
            if weights_change:
                all_gather_params(w_full, self.slot._w_scratch, self.group)


class PeerZeroAdamW:
    """ZeroAdamW with the two collectives as SM kernels over NVLink peer memory
    (coat_zero_step_p2p) instead of NCCL: the gradient and
    both weight buffers live in torch symmetric memory, so every rank maps
    every other rank's copy.  Per step the reduce-scatter reads the peers'
    gradient shards in place (P2P loads summed in rank order, or NVLink-SHARP
    multimem.ld_reduce when the platform gives a multicast address and the
    wire is fp32), K1 steps the shard, and the new shard is stored straight
    into every rank's next-weight buffer (P2P or multimem.st) -- chunk by
    chunk, so the NVLink traffic overlaps the step.  The weights are
    double-buffered: ``weights`` is the current buffer, the step writes the
    other one and the commit flips them -- unless the OR of the ranks' error
    words says the reference's step would have thrown before touching the
    parameters (optimizer.cpp:101-114).

    Usage: write this rank's gradients into ``grad`` (fp32, or bf16 with
    ``grad_dtype=torch.bfloat16`` for the half-width wire), call ``step()``,
    read the parameters from ``weights``."""

    def __init__(self, shapes: Sequence[Sequence[int]], cfg: coatsim.AdamWConfig | None = None, group=None,
                 device=None, grad_dtype: torch.dtype = torch.float32, multicast: bool = True, chunk: int = 0):
        import ctypes as C

        import torch.distributed._symmetric_memory as symm_mem
        if grad_dtype not in (torch.float32, torch.bfloat16):
            raise coatsim.InvalidSpec("PeerZeroAdamW: gradients are float32 or bfloat16")
        self.group = group if group is not None else dist.group.WORLD
        self.world_size, self.rank = _world(self.group)
        self.layout = FlatLayout.build(shapes, self.world_size)
        self.lo, self.hi = self.layout.shard(self.rank)
        self.cfg = cfg or coatsim.AdamWConfig()
        self.chunk = int(chunk)
        device = torch.device(device or "cuda", torch.cuda.current_device()) if not isinstance(device, torch.device) \
            else device
        n = self.layout.total
        self.grad = symm_mem.empty(n, dtype=grad_dtype, device=device)
        self._w = [symm_mem.empty(n, dtype=torch.float32, device=device) for _ in range(2)]
        self._w[0].zero_()
        name = self.group.group_name
        self._hg = symm_mem.rendezvous(self.grad, name)
        hw = [symm_mem.rendezvous(w, name) for w in self._w]
        P = C.c_void_p * self.world_size
        self._g_peers = P(*self._hg.buffer_ptrs)
        self._w_peers = [P(*h.buffer_ptrs) for h in hw]
        use_mc = multicast and grad_dtype == torch.float32
        self._g_mc = (self._hg.multicast_ptr or None) if use_mc else None
        self._w_mc = [(h.multicast_ptr or None) if multicast else None for h in hw]
        self._g_dtype = 0 if grad_dtype == torch.float32 else 1
        self._cur = 0
        self.slot = coatsim.make_slot([self.hi - self.lo], device=device)
        self.g_shard = torch.empty(self.hi - self.lo, dtype=torch.float32, device=device)

    @property
    def weights(self) -> torch.Tensor:
        return self._w[self._cur]

    @property
    def uses_multicast(self) -> bool:
        return self._g_mc is not None

    @property
    def step_count(self) -> int:
        return self.slot.step

    def step(self) -> None:
        import ctypes as C
        L = _lib.lib
        slot, nxt = self.slot, 1 - self._cur
        # every rank's gradients (and the previous step's weight stores) are
        # complete before any rank reads them
        self._hg.barrier()
        mi, vi = slot._m[slot._cm], slot._v[slot._cv]
        mo, vo = slot._m[1 - slot._cm], slot._v[1 - slot._cv]
        slot._flags.t.zero_()
        c = self.cfg.c_struct()
        coatsim._check(L.coat_zero_step_p2p(
            self._g_peers, self._g_mc, self._g_dtype, self._w_peers[nxt], self._w_mc[nxt],
            self._w[self._cur].data_ptr(), self._w[nxt].data_ptr(), self.layout.total, GROUP, mi.c_struct(),
            vi.c_struct(), mo.c_struct(), vo.c_struct(), C.byref(c), slot.step + 1, self.g_shard.data_ptr(),
            slot._flags.ptr, self.rank, self.world_size, self.chunk, coatsim._stream()))
        # the OR of the error words; also the point after which every rank's
        # stores into this rank's next-weight buffer have landed
        flags = _all_flags(slot._flags.t, self.group)
        if not (flags & (_lib.FLAG_NONFINITE_GRAD | _lib.FLAG_CONTRACT)):
            self._cur = nxt
        coatsim._step_commit(None, slot, flags)
