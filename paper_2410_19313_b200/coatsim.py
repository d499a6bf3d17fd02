"""Host-side mirror of the reference's ``proj/core`` operator API on B200.

Same names, argument meaning and error behaviour as coatsim
(/root/reference/proj/core/include/coatsim/*.hpp), so code written against the
reference reads the same here; tensors are CUDA ``torch.Tensor`` s instead of
``coatsim::Tensor`` and every operator runs through the C-ABI of
include/coat.h (libcoat.so, sm_100a).  There is no CPU path.

Mapped surface (reference declaration -> here):

  errors.hpp:8-22                   Error, NonFiniteInput, NonFiniteGradient, ...
  fp8.hpp:47-70                     encode_byte/decode_byte (tensor-wise), round_bf16
  quantize.hpp:14-46                QuantMode, QuantGeometry, QuantizedTensor
  quantize.hpp:70-77                quantize, dequantize, group_scale_max
  expand.hpp:21-71                  ExpandedQuantState, expand_quantize, dequantize_contract
  optimizer.hpp:13-62               AdamWConfig, MomentPolicy, SlotPolicy, OptimizerSlot,
                                    make_slot, step
  optimizer.hpp:72-75               save_slot, load_slot (the reference's file format)
Out of scope: E5M2/DE8 formats, per-block geometry, FP32 scale
dtype, the flow simulator and the memory model -- they raise InvalidSpec.
"""
from __future__ import annotations

import ctypes as C
import enum
import json
import os
from dataclasses import dataclass, field
from typing import Sequence

import torch

from . import _lib

L = _lib.lib
DRE_GROUP = 128  # optimizer-state group


# --------------------------------------------------------------- errors ----
class Error(RuntimeError):
    """coatsim::Error (errors.hpp:8-10)."""


class NonFiniteInput(Error): pass
class NonFiniteGradient(Error): pass
class OutOfRange(Error): pass
class GeometryMismatch(Error): pass
class ShapeMismatch(Error): pass
class AllZeroGroup(Error): pass
class InvalidSpec(Error): pass
class IoError(Error): pass
class BadMagic(Error): pass
class CudaError(Error): pass
class NcclError(Error): pass


_EXC = {1: ShapeMismatch, 2: GeometryMismatch, 3: NonFiniteInput, 4: NonFiniteGradient,
        5: InvalidSpec, 6: CudaError, 7: NcclError, 8: OutOfRange, 9: AllZeroGroup,
        10: IoError, 11: BadMagic}


def _check(status: int) -> None:
    if status != _lib.COAT_OK:
        raise _EXC.get(status, Error)(L.coat_last_error().decode() or _lib.STATUS_NAMES.get(status))


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


class _Flags:
    """A device error word; .raise_if_set() synchronizes and raises like the reference."""

    def __init__(self, device):
        self.t = torch.zeros(1, dtype=torch.int32, device=device)

    @property
    def ptr(self) -> int:
        return self.t.data_ptr()

    def value(self) -> int:
        return int(self.t.item()) & 0xFFFFFFFF

    def raise_if_set(self, what: str) -> None:
        v = self.value()
        if v:
            _check_flags(v, what)


def _check_flags(v: int, what: str) -> None:
    st = L.coat_flags_to_status(v)
    if st:
        raise _EXC[st](f"{what}: non-finite values (flags=0x{v:x})")


def _as_device_input(x: torch.Tensor, what: str) -> tuple[torch.Tensor, int]:
    if not isinstance(x, torch.Tensor) or not x.is_cuda:
        raise InvalidSpec(f"{what}: expected a CUDA tensor")
    if x.dtype == torch.float32:
        dt = 0
    elif x.dtype == torch.bfloat16:
        dt = 1
    else:
        raise InvalidSpec(f"{what}: dtype must be float32 or bfloat16")
    if x.numel() == 0 or any(d <= 0 for d in x.shape):
        raise InvalidSpec("tensor dimensions must be positive")
    return x.contiguous(), dt


# ---------------------------------------------------------------- codec ----
class Fp8Tag(enum.IntEnum):
    E4M3 = 0
    E5M2 = 1
    DE8 = 2


@dataclass(frozen=True)
class Fp8Format:
    """fp8.hpp:26-38.  Only E4M3 is on the hot path."""
    tag: Fp8Tag
    delta_max: float
    delta_min: float
    mantissa_bits: int
    exponent_bits: int

    @staticmethod
    def e4m3() -> "Fp8Format":
        return _E4M3

    def dynamic_range(self) -> float:
        return self.delta_max / self.delta_min


_E4M3 = Fp8Format(Fp8Tag.E4M3, 448.0, 2.0 ** -9, 3, 4)


def _require_e4m3(fmt: Fp8Format | None) -> None:
    if fmt is not None and fmt.tag != Fp8Tag.E4M3:
        raise InvalidSpec("only the E4M3 format is implemented on the B200 path")


def encode_e4m3(x: torch.Tensor) -> torch.Tensor:
    """encode_byte(x, e4m3) elementwise (fp8.cpp:150-156)."""
    x = x.contiguous().float()
    out = torch.empty(x.shape, dtype=torch.uint8, device=x.device)
    fl = _Flags(x.device)
    _check(L.coat_encode_e4m3(x.data_ptr(), out.data_ptr(), x.numel(), fl.ptr, _stream()))
    fl.raise_if_set("encode")
    return out


def decode_e4m3(codes: torch.Tensor) -> torch.Tensor:
    """decode_byte(code, e4m3) elementwise (fp8.cpp:145-148)."""
    codes = codes.contiguous()
    out = torch.empty(codes.shape, dtype=torch.float32, device=codes.device)
    _check(L.coat_decode_e4m3(codes.data_ptr(), out.data_ptr(), codes.numel(), _stream()))
    return out


# ------------------------------------------------------------ quantizer ----
class QuantMode(enum.IntEnum):
    PerTensor = 0
    PerGroup = 1
    PerBlock = 2


@dataclass(frozen=True)
class QuantGeometry:
    """quantize.hpp:14-26."""
    mode: QuantMode = QuantMode.PerTensor
    group_size: int = 0
    block_size: int = 0

    @staticmethod
    def per_tensor() -> "QuantGeometry":
        return QuantGeometry(QuantMode.PerTensor, 0, 0)

    @staticmethod
    def per_group(g: int) -> "QuantGeometry":
        return QuantGeometry(QuantMode.PerGroup, int(g), 0)

    @staticmethod
    def per_block(b: int) -> "QuantGeometry":
        return QuantGeometry(QuantMode.PerBlock, 0, int(b))


@dataclass
class QuantizedTensor:
    """quantize.hpp:37-46.  ``scales`` is a bfloat16 tensor (the reference's
    float scales are always BF16-valued, so this is lossless)."""
    codes: torch.Tensor
    scales: torch.Tensor
    geometry: QuantGeometry
    format: Fp8Tag = Fp8Tag.E4M3
    source_shape: tuple = ()

    def numel(self) -> int:
        return self.codes.numel()

    def group_count(self) -> int:
        return self.scales.numel()


def _rows_cols(shape: Sequence[int]) -> tuple[int, int]:
    cols = int(shape[-1]) if len(shape) else 1
    rows = 1
    for d in shape[:-1]:
        rows *= int(d)
    return rows, cols


def _per_tensor_stage1_group(cols: int) -> int:
    """Stage-1 group of the Group Scaling amax for per-tensor quantization:
    1x128 when it divides the last dim, else the whole row (any G gives the
    same global max bitwise, test_quantize.cpp:127-146)."""
    return 128 if cols % 128 == 0 else cols


def group_scale_max_device(x: torch.Tensor, group_size: int, want_intermediate: bool = True):
    """Two-stage Group Scaling amax without a host sync: returns
    (intermediate or None, amax_bits int32 device tensor of shape [1])."""
    x, dt = _as_device_input(x, "group_scale_max")
    rows, cols = _rows_cols(x.shape)
    inter = None
    if want_intermediate and group_size > 0 and cols % group_size == 0:
        inter = torch.empty(tuple(x.shape[:-1]) + (cols // group_size,), dtype=torch.float32,
                            device=x.device)
    amax = torch.empty(1, dtype=torch.int32, device=x.device)
    _check(L.coat_group_scale_max(x.data_ptr(), dt, rows, cols, int(group_size), _ptr(inter),
                                  amax.data_ptr(), _stream()))
    return inter, amax


def group_scale_max(x: torch.Tensor, group_size: int):
    """quantize.hpp:77 -> (intermediate tensor, global max as a Python float)."""
    inter, amax = group_scale_max_device(x, group_size)
    g = amax.view(torch.float32).item()
    return inter, g


def quantize(x: torch.Tensor, geometry: QuantGeometry, format: Fp8Format | None = None,
             options=None) -> QuantizedTensor:
    """quantize.hpp:70-71 (E4M3, BF16 scales)."""
    _require_e4m3(format)
    if options is not None and getattr(options, "scale_dtype", "bf16") not in ("bf16", 0):
        raise InvalidSpec("only BF16 scales are implemented on the B200 path")
    x, dt = _as_device_input(x, "quantize")
    rows, cols = _rows_cols(x.shape)
    fl = _Flags(x.device)
    codes = torch.empty(x.shape, dtype=torch.uint8, device=x.device)
    if geometry.mode == QuantMode.PerGroup:
        G = geometry.group_size
        if G <= 0:
            raise GeometryMismatch("per-group: group size must be positive")
        if cols % G != 0:
            raise GeometryMismatch("per-group: last dim not divisible by group size")
        scales = torch.empty(x.numel() // G, dtype=torch.bfloat16, device=x.device)
        _check(L.coat_quantize_per_group(x.data_ptr(), dt, rows, cols, G, codes.data_ptr(),
                                         scales.data_ptr(), fl.ptr, _stream()))
    elif geometry.mode == QuantMode.PerTensor:
        _, amax = group_scale_max_device(x, _per_tensor_stage1_group(cols), want_intermediate=False)
        scales = torch.empty(1, dtype=torch.bfloat16, device=x.device)
        _check(L.coat_quantize_per_tensor(x.data_ptr(), dt, x.numel(), amax.data_ptr(),
                                          codes.data_ptr(), scales.data_ptr(), fl.ptr, _stream()))
    else:
        raise InvalidSpec("per-block geometry is outside the B200 hot path (SURVEY.md 2)")
    fl.raise_if_set("quantize")
    return QuantizedTensor(codes, scales, geometry, Fp8Tag.E4M3, tuple(x.shape))


def quantize_batch(items: Sequence[tuple[torch.Tensor, QuantGeometry]]) -> list[QuantizedTensor]:
    """MGAQ of a layer in one launch (coat_quantize_batch): the same results as
    ``[quantize(x, g) for x, g in items]`` (per-group or per-tensor with Group
    Scaling amax).  Up to 16 items; inputs 32-byte aligned with numel % 16 == 0."""
    if not items:
        return []
    if len(items) > 16:
        raise InvalidSpec("quantize_batch: at most 16 items")
    arr = (_lib.MgaqItemC * len(items))()
    out, keep = [], []
    dev = None
    for i, (x, geo) in enumerate(items):
        x, dt = _as_device_input(x, "quantize_batch")
        dev = x.device
        rows, cols = _rows_cols(x.shape)
        codes = torch.empty(x.shape, dtype=torch.uint8, device=x.device)
        if geo.mode == QuantMode.PerGroup:
            G = geo.group_size
            if G <= 0 or cols % G != 0:
                raise GeometryMismatch("per-group: last dim not divisible by group size")
            scales = torch.empty(x.numel() // G, dtype=torch.bfloat16, device=x.device)
        elif geo.mode == QuantMode.PerTensor:
            G = 0
            scales = torch.empty(1, dtype=torch.bfloat16, device=x.device)
        else:
            raise InvalidSpec("per-block geometry is outside the B200 hot path (SURVEY.md 2)")
        arr[i] = _lib.MgaqItemC(x.data_ptr(), dt, 0, rows, cols, G, codes.data_ptr(), scales.data_ptr(), None)
        keep.append(x)
        out.append(QuantizedTensor(codes, scales, geo, Fp8Tag.E4M3, tuple(x.shape)))
    fl = _Flags(dev)
    _check(L.coat_quantize_batch(arr, len(items), fl.ptr, _stream()))
    fl.raise_if_set("quantize")
    return out


def dequantize(q: QuantizedTensor, out_dtype: torch.dtype = torch.float32) -> torch.Tensor:
    """quantize.hpp:72 (fp32 like the reference; bf16 optional)."""
    odt = 0 if out_dtype == torch.float32 else 1
    out = torch.empty(q.source_shape, dtype=out_dtype, device=q.codes.device)
    rows, cols = _rows_cols(q.source_shape)
    if q.geometry.mode == QuantMode.PerGroup:
        _check(L.coat_dequantize_per_group(q.codes.data_ptr(), q.scales.data_ptr(), rows, cols,
                                           q.geometry.group_size, out.data_ptr(), odt, _stream()))
    elif q.geometry.mode == QuantMode.PerTensor:
        _check(L.coat_dequantize_per_tensor(q.codes.data_ptr(), q.scales.data_ptr(), q.numel(),
                                            out.data_ptr(), odt, _stream()))
    else:
        raise InvalidSpec("per-block geometry is outside the B200 hot path (SURVEY.md 2)")
    return out


def quantization_error(x: torch.Tensor, geometry: QuantGeometry, format=None) -> float:
    """quantize.hpp:80-81: MSE between x and dequantize(quantize(x))."""
    back = dequantize(quantize(x, geometry, format))
    return float(((back.double() - x.double()) ** 2).mean().item())


# ------------------------------------------------------ range expansion ----
class MomentBuffers:
    """Device storage of one E4M3+DRE moment (codes, bf16 scales, k, c)."""

    def __init__(self, npad: int, device):
        ng = npad // DRE_GROUP
        self.npad = npad
        self.codes = torch.empty(npad, dtype=torch.uint8, device=device)
        self.scales = torch.empty(ng, dtype=torch.bfloat16, device=device)
        self.k = torch.empty(ng, dtype=torch.float32, device=device)
        self.c = torch.empty(ng, dtype=torch.float32, device=device)

    def c_struct(self) -> _lib.MomentState:
        return _lib.MomentState(self.codes.data_ptr(), self.scales.data_ptr(), self.k.data_ptr(),
                                self.c.data_ptr())

    def clone(self) -> "MomentBuffers":
        b = MomentBuffers.__new__(MomentBuffers)
        b.npad = self.npad
        b.codes, b.scales, b.k, b.c = (t.clone() for t in (self.codes, self.scales, self.k, self.c))
        return b


@dataclass
class ExpandedQuantState:
    """expand.hpp:60-63: per-group (1xG) E4M3 codes + BF16 scales + (k, c)."""
    quantized: QuantizedTensor
    k: torch.Tensor
    c: torch.Tensor

    @property
    def degenerate(self) -> torch.Tensor:   # tensor_io.cpp:172: degenerate = (k == 1)
        return self.k == 1.0

    @staticmethod
    def _from_buffers(b: MomentBuffers, shape) -> "ExpandedQuantState":
        q = QuantizedTensor(b.codes, b.scales, QuantGeometry.per_group(DRE_GROUP), Fp8Tag.E4M3,
                            tuple(shape))
        return ExpandedQuantState(q, b.k, b.c)

    def _buffers(self) -> MomentBuffers:
        b = MomentBuffers.__new__(MomentBuffers)
        b.npad = self.quantized.codes.numel()
        b.codes, b.scales, b.k, b.c = self.quantized.codes, self.quantized.scales, self.k, self.c
        return b


def _check_dre_group(group_size: int) -> None:
    if group_size != DRE_GROUP:
        raise InvalidSpec("the B200 DRE kernels implement the 1x128 optimizer group only")


def expand_quantize(x: torch.Tensor, group_size: int = DRE_GROUP, format: Fp8Format | None = None,
                    options=None) -> ExpandedQuantState:
    """expand.hpp:67-68 on a (flattened) fp32 tensor."""
    _require_e4m3(format)
    if not isinstance(x, torch.Tensor) or not x.is_cuda or x.dtype != torch.float32:
        raise InvalidSpec("expand_quantize: expected a float32 CUDA tensor")
    n = x.numel()
    if group_size <= 0 or n % group_size != 0:
        raise GeometryMismatch("per-group: last dim not divisible by group size")
    _check_dre_group(group_size)
    x = x.contiguous()
    b = MomentBuffers(n, x.device)
    fl = _Flags(x.device)
    _check(L.coat_expand_quantize(x.data_ptr(), n, group_size, b.c_struct(), fl.ptr, _stream()))
    fl.raise_if_set("expand_quantize")
    return ExpandedQuantState._from_buffers(b, x.shape)


def dequantize_contract(state: ExpandedQuantState) -> torch.Tensor:
    """expand.hpp:71."""
    q = state.quantized
    out = torch.empty(q.codes.numel(), dtype=torch.float32, device=q.codes.device)
    fl = _Flags(out.device)
    _check(L.coat_dequantize_contract(state._buffers().c_struct(), out.numel(), DRE_GROUP,
                                      out.data_ptr(), fl.ptr, _stream()))
    fl.raise_if_set("dequantize_contract")
    return out.view(q.source_shape) if out.numel() == _numel(q.source_shape) else out


def _numel(shape) -> int:
    n = 1
    for d in shape:
        n *= int(d)
    return n


# ------------------------------------------------------------ optimizer ----
@dataclass
class AdamWConfig:
    """optimizer.hpp:13-20."""
    beta1: float = 0.9
    beta2: float = 0.999
    lr: float = 1e-3
    weight_decay: float = 0.0
    eps: float = 1e-8
    step: int = 0

    def c_struct(self) -> _lib.AdamWConfigC:
        return _lib.AdamWConfigC(self.beta1, self.beta2, self.lr, self.weight_decay, self.eps)


class StateFormat(enum.IntEnum):
    FP32 = 0
    E4M3 = 1
    E5M2 = 2
    DE8 = 3


@dataclass
class MomentPolicy:
    """optimizer.hpp:30-34; the B200 path implements {E4M3, expand, 128}."""
    format: StateFormat = StateFormat.E4M3
    expand: bool = True
    group_size: int = DRE_GROUP


@dataclass
class SlotPolicy:
    first: MomentPolicy = field(default_factory=MomentPolicy)
    second: MomentPolicy = field(default_factory=MomentPolicy)


def _check_policy(p: SlotPolicy) -> None:
    for mp in (p.first, p.second):
        if mp.format != StateFormat.E4M3 or not mp.expand:
            raise InvalidSpec("the B200 optimizer implements the {E4M3, expand} policy only")
        _check_dre_group(mp.group_size)


class OptimizerSlot:
    """optimizer.hpp:46-52.  Holds two buffer sets per moment (ping-pong) so a
    failed step commits exactly what the reference commits."""

    def __init__(self, shape, policy: SlotPolicy, device):
        self.shape = tuple(int(d) for d in shape)
        self.policy = policy
        self.step = 0
        n = _numel(self.shape)
        npad = -(-n // DRE_GROUP) * DRE_GROUP
        self._m = [MomentBuffers(npad, device), MomentBuffers(npad, device)]
        self._v = [MomentBuffers(npad, device), MomentBuffers(npad, device)]
        self._cm = 0
        self._cv = 0
        self._w_scratch = None
        self._flags = _Flags(device)

    @property
    def m(self) -> ExpandedQuantState:
        return ExpandedQuantState._from_buffers(self._m[self._cm], (self._m[0].npad,))

    @property
    def v(self) -> ExpandedQuantState:
        return ExpandedQuantState._from_buffers(self._v[self._cv], (self._v[0].npad,))

    def load_state(self, m: dict, v: dict, step: int) -> None:
        """Overwrite the current state from host/device arrays (codes, scales, k, c)."""
        for buf, src in ((self._m[self._cm], m), (self._v[self._cv], v)):
            buf.codes.copy_(torch.as_tensor(src["codes"]))
            sc = torch.as_tensor(src["scales"])
            buf.scales.copy_(sc if sc.dtype == torch.bfloat16 else sc.to(torch.float32).to(torch.bfloat16))
            buf.k.copy_(torch.as_tensor(src["k"]))
            buf.c.copy_(torch.as_tensor(src["c"]))
        self.step = int(step)


def make_slot(shape, policy: SlotPolicy | None = None, device="cuda") -> OptimizerSlot:
    """optimizer.hpp:54 (optimizer.cpp:90-99)."""
    policy = policy or SlotPolicy()
    _check_policy(policy)
    shape = [int(d) for d in shape]
    if any(d <= 0 for d in shape):
        raise InvalidSpec("tensor dimensions must be positive")
    slot = OptimizerSlot(shape, policy, torch.device(device))
    n = _numel(shape)
    _check(L.coat_make_slot(n, DRE_GROUP, slot._m[0].c_struct(), slot._v[0].c_struct(), _stream()))
    return slot


def _step_launch(params: torch.Tensor, grads: torch.Tensor, slot: OptimizerSlot, cfg: AdamWConfig) -> None:
    """Validate (before any mutation, like optimizer.cpp:102-104) and launch the
    fused kernel into the slot's spare buffers; nothing is committed yet."""
    if tuple(params.shape) != slot.shape:
        raise ShapeMismatch("step: params do not match slot shape")
    if tuple(grads.shape) != tuple(params.shape):
        raise ShapeMismatch("step: shape mismatch")
    if params.dtype != torch.float32 or grads.dtype != torch.float32:
        raise InvalidSpec("step: params and grads must be float32")
    if not params.is_contiguous():
        raise InvalidSpec("step: params must be contiguous")
    grads = grads.contiguous()
    n = params.numel()
    if slot._w_scratch is None or slot._w_scratch.numel() != n:
        slot._w_scratch = torch.empty_like(params)
    t = slot.step + 1
    mi, vi = slot._m[slot._cm], slot._v[slot._cv]
    mo, vo = slot._m[1 - slot._cm], slot._v[1 - slot._cv]
    slot._flags.t.zero_()
    c = cfg.c_struct()
    _check(L.coat_adamw_dre_step(params.data_ptr(), slot._w_scratch.data_ptr(), grads.data_ptr(),
                                 n, DRE_GROUP, mi.c_struct(), vi.c_struct(), mo.c_struct(),
                                 vo.c_struct(), C.byref(c), t, slot._flags.ptr, _stream()))


def _step_commit(params: torch.Tensor | None, slot: OptimizerSlot, flags: int) -> None:
    """Commit a launched step exactly as the reference would have (optimizer.cpp:101-114):

    * NonFiniteGradient (optimizer.cpp:104): nothing is mutated.
    * NonFiniteInput from unpack (contract): nothing is mutated.
    * NonFiniteInput from pack_moment(m): params updated, slot unchanged.
    * NonFiniteInput from pack_moment(v): params and slot.m updated, v and step not.
    params=None: the caller publishes slot._w_scratch itself (ZeRO all-gather).
    """
    if flags & _lib.FLAG_NONFINITE_GRAD:
        raise NonFiniteGradient("step: gradient has non-finite values")
    if flags & _lib.FLAG_CONTRACT:
        raise NonFiniteInput("contract: tensor has non-finite values")
    if params is not None:
        params.copy_(slot._w_scratch)
    if flags & _lib.FLAG_PACK_M:
        raise NonFiniteInput("expand_quantize: tensor has non-finite values")
    slot._cm = 1 - slot._cm
    if flags & _lib.FLAG_PACK_V:
        raise NonFiniteInput("expand_quantize: tensor has non-finite values")
    slot._cv = 1 - slot._cv
    slot.step = slot.step + 1


def step(params: torch.Tensor, grads: torch.Tensor, slot: OptimizerSlot, cfg: AdamWConfig,
         check: bool = True) -> None:
    """optimizer.hpp:58: one fused kernel (K1), then commit like the reference
    (see _step_commit for the error semantics)."""
    _step_launch(params, grads, slot, cfg)
    _step_commit(params, slot, slot._flags.value() if check else 0)


# --------------------------------------------- fused producers + MGAQ (a17) ----
def rmsnorm_quantize(x: torch.Tensor, w: torch.Tensor, eps: float = 1e-6, return_y: bool = False):
    """The RMSNorm block of the COAT forward (flow.cpp:546-549): returns
    (Q_g16(x), Q_t(rmsnorm(DQ(Q_g16(x)), w)), rms per row[, y]) -- the
    rmsnorm1.in / qkv.in records, bit-identical to the reference's tape."""
    x, dt = _as_device_input(x, "rmsnorm_quantize")
    rows, h = _rows_cols(x.shape)
    w = w.to(device=x.device, dtype=torch.float32).contiguous()
    if w.numel() != h:
        raise ShapeMismatch("rmsnorm_quantize: weight must have h elements")
    dev = x.device
    xc = torch.empty(x.shape, dtype=torch.uint8, device=dev)
    xs = torch.empty(x.numel() // 16, dtype=torch.bfloat16, device=dev)
    yc = torch.empty(x.shape, dtype=torch.uint8, device=dev)
    ys = torch.empty(1, dtype=torch.bfloat16, device=dev)
    rms = torch.empty(rows, dtype=torch.float32, device=dev)
    amax = torch.empty(1, dtype=torch.int32, device=dev)
    y = torch.empty(x.shape, dtype=torch.float32, device=dev) if return_y else None
    fl = _Flags(dev)
    _check(L.coat_rmsnorm_quant(x.data_ptr(), dt, rows, h, w.data_ptr(), eps, xc.data_ptr(), xs.data_ptr(),
                                yc.data_ptr(), ys.data_ptr(), _ptr(y), rms.data_ptr(), amax.data_ptr(), fl.ptr,
                                _stream()))
    fl.raise_if_set("rmsnorm_quantize")
    qx = QuantizedTensor(xc, xs, QuantGeometry.per_group(16), Fp8Tag.E4M3, tuple(x.shape))
    qy = QuantizedTensor(yc, ys, QuantGeometry.per_tensor(), Fp8Tag.E4M3, tuple(x.shape))
    return (qx, qy, rms, y) if return_y else (qx, qy, rms)


def silu_mul_quantize(gate: torch.Tensor, up: torch.Tensor, return_prod: bool = False):
    """The SiLU*mul block (flow.cpp:603-612): returns the silu.in, mul.in.silu,
    mul.in.up (per-group 1x16) and down.in (per-tensor) records[, prod]."""
    gate, dt = _as_device_input(gate, "silu_mul_quantize")
    up, dt2 = _as_device_input(up, "silu_mul_quantize")
    if up.shape != gate.shape or dt2 != dt:
        raise ShapeMismatch("silu_mul_quantize: gate and up must match in shape and dtype")
    rows, cols = _rows_cols(gate.shape)
    dev = gate.device
    mk = lambda: (torch.empty(gate.shape, dtype=torch.uint8, device=dev),
                  torch.empty(gate.numel() // 16, dtype=torch.bfloat16, device=dev))
    (gc, gs), (sc, ss), (uc, us) = mk(), mk(), mk()
    pc = torch.empty(gate.shape, dtype=torch.uint8, device=dev)
    ps = torch.empty(1, dtype=torch.bfloat16, device=dev)
    amax = torch.empty(1, dtype=torch.int32, device=dev)
    p = torch.empty(gate.shape, dtype=torch.float32, device=dev) if return_prod else None
    fl = _Flags(dev)
    _check(L.coat_silu_mul_quant(gate.data_ptr(), up.data_ptr(), dt, rows, cols, gc.data_ptr(), gs.data_ptr(),
                                 sc.data_ptr(), ss.data_ptr(), uc.data_ptr(), us.data_ptr(), pc.data_ptr(),
                                 ps.data_ptr(), _ptr(p), amax.data_ptr(), fl.ptr, _stream()))
    fl.raise_if_set("silu_mul_quantize")
    g16, shp = QuantGeometry.per_group(16), tuple(gate.shape)
    out = (QuantizedTensor(gc, gs, g16, Fp8Tag.E4M3, shp), QuantizedTensor(sc, ss, g16, Fp8Tag.E4M3, shp),
           QuantizedTensor(uc, us, g16, Fp8Tag.E4M3, shp),
           QuantizedTensor(pc, ps, QuantGeometry.per_tensor(), Fp8Tag.E4M3, shp))
    return out + (p,) if return_prod else out


# -------------------------------------------------- backward-side MGAQ pieces ----
def used_values_transposed(q: QuantizedTensor, out_dtype: torch.dtype = torch.float32,
                           return_codes: bool = False):
    """SavedActivation::used_values_transposed (flow.cpp:360-395): the
    dequantized transpose [cols, rows] of a 2-D FP8 save (wgrad operand);
    per-group scales follow the original row-major grouping."""
    if q.geometry.mode not in (QuantMode.PerGroup, QuantMode.PerTensor):
        raise InvalidSpec("per-block geometry is outside the B200 hot path (SURVEY.md 2)")
    rows, cols = _rows_cols(q.source_shape)
    G = q.geometry.group_size if q.geometry.mode == QuantMode.PerGroup else 0
    dev = q.codes.device
    out = torch.empty(cols, rows, dtype=out_dtype, device=dev)
    ct = torch.empty(cols, rows, dtype=torch.uint8, device=dev) if return_codes else None
    _check(L.coat_transpose_dequantize(q.codes.data_ptr(), q.scales.data_ptr(), rows, cols, G, out.data_ptr(),
                                       0 if out_dtype == torch.float32 else 1, _ptr(ct), _stream()))
    return (out, ct) if return_codes else out


def requantize_cached(x: torch.Tensor, cached_scale: torch.Tensor, out_dtype: torch.dtype = torch.float32,
                      return_codes: bool = False):
    """requantize_cached (flow.cpp:487-495): decode(encode(x / s)) * s against
    the per-tensor BF16 scale cached in the forward (``cached_scale``, 1 element)."""
    x, dt = _as_device_input(x, "requantize_cached")
    s = cached_scale.to(device=x.device, dtype=torch.bfloat16).reshape(1).contiguous()
    out = torch.empty(x.shape, dtype=out_dtype, device=x.device)
    codes = torch.empty(x.shape, dtype=torch.uint8, device=x.device) if return_codes else None
    fl = _Flags(x.device)
    _check(L.coat_requantize_cached(x.data_ptr(), dt, x.numel(), s.data_ptr(), out.data_ptr(),
                                    0 if out_dtype == torch.float32 else 1, _ptr(codes), fl.ptr, _stream()))
    fl.raise_if_set("requantize_cached")
    return (out, codes) if return_codes else out


class WeightOperandCache:
    """DecoderLayer::weight_operand + start_accumulation_cycle (flow.cpp:499-530):
    a master weight is quantized per-tensor (Group Scaling amax) at most once
    per gradient-accumulation cycle; later uses in the cycle reuse the codes."""

    def __init__(self):
        self._cache: dict = {}
        self.weight_scale_computations = 0

    def start_accumulation_cycle(self) -> None:
        self._cache.clear()

    def operand(self, name: str, master: torch.Tensor) -> QuantizedTensor:
        q = self._cache.get(name)
        if q is None:
            q = quantize(master, QuantGeometry.per_tensor())
            self._cache[name] = q
            self.weight_scale_computations += 1
        return q


# ------------------------------------------------------- slot checkpoints ----
def save_slot(path: str, slot: OptimizerSlot, cfg: AdamWConfig) -> None:
    """optimizer.hpp:74 (optimizer.cpp:196-252): the reference's binary slot
    format, byte-identical to what coatsim::save_slot writes for the same state."""
    shape = (C.c_int64 * len(slot.shape))(*slot.shape)
    c = cfg.c_struct()
    _check(L.coat_save_slot(os.fsencode(path), shape, len(slot.shape), DRE_GROUP,
                            slot._m[slot._cm].c_struct(), slot._v[slot._cv].c_struct(), C.byref(c),
                            slot.step, _stream()))


def load_slot(path: str, device="cuda") -> tuple[OptimizerSlot, AdamWConfig]:
    """optimizer.hpp:75: load a slot written by the reference (or save_slot);
    InvalidSpec unless the policy is {E4M3, expand, 128} for both moments."""
    try:
        with open(path, "rb") as f:
            n = int.from_bytes(f.read(4), "little")
            header = json.loads(f.read(n))
        shape = [int(d) for d in header["shape"]]
    except (OSError, ValueError, KeyError) as e:
        raise IoError(f"load_slot: cannot read header of {path}: {e}") from None
    slot = OptimizerSlot(shape, SlotPolicy(), torch.device(device))
    cs = (C.c_int64 * len(shape))(*shape)
    cfg_c = _lib.AdamWConfigC()
    step = C.c_int64(0)
    _check(L.coat_load_slot(os.fsencode(path), cs, len(shape), DRE_GROUP, slot._m[slot._cm].c_struct(),
                            slot._v[slot._cv].c_struct(), C.byref(cfg_c), C.byref(step), _stream()))
    slot.step = int(step.value)
    cfg = AdamWConfig(beta1=cfg_c.beta1, beta2=cfg_c.beta2, lr=cfg_c.lr, weight_decay=cfg_c.weight_decay,
                      eps=cfg_c.eps, step=slot.step)
    return slot, cfg


# ------------------------------------------------------------ FP8 linear ----
# The reference's linear (flow.cpp:21-46) has no public entry point; these
# follow its semantics on tcgen05 (gemm_tcgen05.cu).

def _per_tensor(q: QuantizedTensor, what: str) -> None:
    if q.geometry.mode != QuantMode.PerTensor or len(q.source_shape) != 2:
        raise InvalidSpec(f"{what}: expected a 2-D per-tensor QuantizedTensor")


def decode_e4m3_bf16(codes: torch.Tensor) -> torch.Tensor:
    """decode_byte of every code as bfloat16 (exact)."""
    codes = codes.contiguous()
    out = torch.empty(codes.shape, dtype=torch.bfloat16, device=codes.device)
    _check(L.coat_decode_e4m3_bf16(codes.data_ptr(), out.data_ptr(), codes.numel(), _stream()))
    return out


def fp8_linear(qx: QuantizedTensor, qw: QuantizedTensor) -> torch.Tensor:
    """y = matmul(DQ(Q_t(x)), DQ(Q_t(W))) (flow.cpp:21-33, 548-552); W is (K, N)."""
    _per_tensor(qx, "fp8_linear")
    _per_tensor(qw, "fp8_linear")
    (M, K), (K2, N) = qx.source_shape, qw.source_shape
    if K != K2:
        raise ShapeMismatch("fp8_linear: inner dimensions differ")
    y = torch.empty(M, N, dtype=torch.float32, device=qx.codes.device)
    _check(L.coat_fp8_linear_fwd(qx.codes.data_ptr(), qx.scales.data_ptr(), qw.codes.data_ptr(),
                                 qw.scales.data_ptr(), M, K, N, y.data_ptr(), _stream()))
    return y


def fp8_linear_q16(qx: QuantizedTensor, qw: QuantizedTensor, return_y: bool = False):
    """quantize(fp8_linear(qx, qw), per_group(16)) with the quantizer in the
    GEMM epilogue: the product never reaches HBM unless
    return_y (then also the fp32 y)."""
    _per_tensor(qx, "fp8_linear_q16")
    _per_tensor(qw, "fp8_linear_q16")
    (M, K), (K2, N) = qx.source_shape, qw.source_shape
    if K != K2:
        raise ShapeMismatch("fp8_linear_q16: inner dimensions differ")
    if N % 16:
        raise GeometryMismatch("per-group: last dim not divisible by group size")
    dev = qx.codes.device
    yc = torch.empty(M, N, dtype=torch.uint8, device=dev)
    ys = torch.empty(M * N // 16, dtype=torch.bfloat16, device=dev)
    y = torch.empty(M, N, dtype=torch.float32, device=dev) if return_y else None
    fl = _Flags(dev)
    _check(L.coat_fp8_linear_fwd_q16(qx.codes.data_ptr(), qx.scales.data_ptr(), qw.codes.data_ptr(),
                                     qw.scales.data_ptr(), M, K, N, yc.data_ptr(), ys.data_ptr(), _ptr(y), fl.ptr,
                                     _stream()))
    fl.raise_if_set("fp8_linear_q16")
    q = QuantizedTensor(yc, ys, QuantGeometry.per_group(16), Fp8Tag.E4M3, (M, N))
    return (q, y) if return_y else q


def fp8_upgate_silu(qx: QuantizedTensor, qw_gate: QuantizedTensor, qw_up: QuantizedTensor,
                    return_fp32: bool = False):
    """The MLP's gate/up projections and the SiLU*mul block (flow.cpp:599-612)
    as ONE tcgen05 GEMM whose epilogue quantizes: returns the silu.in,
    mul.in.silu, mul.in.up (per-group 1x16) and down.in (per-tensor) records
    -- equal to silu_mul_quantize(fp8_linear(qx, qw_gate), fp8_linear(qx,
    qw_up)) -- [, gate, up, prod] (fp32) with return_fp32."""
    for q, what in ((qx, "x"), (qw_gate, "W_gate"), (qw_up, "W_up")):
        _per_tensor(q, f"fp8_upgate_silu {what}")
    (M, H), (H2, I) = qx.source_shape, qw_gate.source_shape
    if H != H2 or tuple(qw_up.source_shape) != (H, I):
        raise ShapeMismatch("fp8_upgate_silu: x (M, H), W_gate and W_up (H, I)")
    if I % 16:
        raise GeometryMismatch("per-group: last dim not divisible by group size")
    dev = qx.codes.device
    mk = lambda: (torch.empty(M, I, dtype=torch.uint8, device=dev),
                  torch.empty(M * I // 16, dtype=torch.bfloat16, device=dev))
    (gc, gs), (sc, ss), (uc, us) = mk(), mk(), mk()
    pc = torch.empty(M, I, dtype=torch.uint8, device=dev)
    ps = torch.empty(1, dtype=torch.bfloat16, device=dev)
    amax = torch.empty(1, dtype=torch.int32, device=dev)
    f32 = (lambda: torch.empty(M, I, dtype=torch.float32, device=dev)) if return_fp32 else (lambda: None)
    g, u, p = f32(), f32(), f32()
    fl = _Flags(dev)
    _check(L.coat_fp8_upgate_silu_quant(qx.codes.data_ptr(), qx.scales.data_ptr(), qw_gate.codes.data_ptr(),
                                        qw_gate.scales.data_ptr(), qw_up.codes.data_ptr(), qw_up.scales.data_ptr(),
                                        M, H, I, gc.data_ptr(), gs.data_ptr(), sc.data_ptr(), ss.data_ptr(),
                                        uc.data_ptr(), us.data_ptr(), pc.data_ptr(), ps.data_ptr(), _ptr(g), _ptr(u),
                                        _ptr(p), amax.data_ptr(), fl.ptr, _stream()))
    fl.raise_if_set("fp8_upgate_silu")
    g16, shp = QuantGeometry.per_group(16), (M, I)
    out = (QuantizedTensor(gc, gs, g16, Fp8Tag.E4M3, shp), QuantizedTensor(sc, ss, g16, Fp8Tag.E4M3, shp),
           QuantizedTensor(uc, us, g16, Fp8Tag.E4M3, shp),
           QuantizedTensor(pc, ps, QuantGeometry.per_tensor(), Fp8Tag.E4M3, shp))
    return out + (g, u, p) if return_fp32 else out


def linear_dgrad(dy: torch.Tensor, qw: QuantizedTensor, w_dec: torch.Tensor | None = None) -> torch.Tensor:
    """dX = bf16(dY . W_used^T) (flow.cpp:636); dY is BF16 and not quantized."""
    _per_tensor(qw, "linear_dgrad")
    K, N = qw.source_shape
    M = dy.shape[0]
    if tuple(dy.shape) != (M, N) or dy.dtype != torch.bfloat16:
        raise ShapeMismatch("linear_dgrad: dY must be bf16 (M, N)")
    w_dec = decode_e4m3_bf16(qw.codes) if w_dec is None else w_dec
    dx = torch.empty(M, K, dtype=torch.bfloat16, device=dy.device)
    _check(L.coat_linear_bwd_dgrad(dy.contiguous().data_ptr(), w_dec.data_ptr(), qw.scales.data_ptr(), M, K, N,
                                   dx.data_ptr(), _stream()))
    return dx


def linear_wgrad(qx: QuantizedTensor, dy: torch.Tensor, x_dec: torch.Tensor | None = None) -> torch.Tensor:
    """dW = X_used^T . dY (flow.cpp:637 with used_values_transposed, 360-395)."""
    _per_tensor(qx, "linear_wgrad")
    M, K = qx.source_shape
    N = dy.shape[1]
    if tuple(dy.shape) != (M, N) or dy.dtype != torch.bfloat16:
        raise ShapeMismatch("linear_wgrad: dY must be bf16 (M, N)")
    x_dec = decode_e4m3_bf16(qx.codes) if x_dec is None else x_dec
    dw = torch.empty(K, N, dtype=torch.float32, device=dy.device)
    _check(L.coat_linear_bwd_wgrad(x_dec.data_ptr(), qx.scales.data_ptr(), dy.contiguous().data_ptr(), M, K, N,
                                   dw.data_ptr(), _stream()))
    return dw


def set_fallback_counter(counter: torch.Tensor | None) -> None:
    """Diagnostics: count literal-formula fallbacks of the DRE kernels."""
    _check(L.coat_set_fallback_counter(None if counter is None else counter.data_ptr()))
