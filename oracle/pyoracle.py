"""oracle/pyoracle.py -- TEST INFRASTRUCTURE ONLY.

numpy/ctypes front-end for the two CPU checkers built by oracle/Makefile:

* ``Oracle("port")``      -> oracle/_build/liboracle.so   (my C restatement, coat_oracle.c)
* ``Oracle("reference")`` -> oracle/_ref/libcoatsim_ref.so (the unmodified reference core
                             compiled out-of-tree + the ref_shim.cpp C wrapper)

Both expose the same methods with the same array conventions, so tests can run
one check against either (and pin the port against the reference).  Only
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference legs
may import this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_LIB = os.path.join(HERE, "_build", "liboracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libcoatsim_ref.so")

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_i64 = C.c_int64
_f = C.c_float


def build(quiet: bool = True) -> None:
    """Build the checkers (the reference only where /root/reference exists)."""
    out = subprocess.run(["make", "-C", HERE, "-j8"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)


def available(kind: str) -> bool:
    return os.path.exists(PORT_LIB if kind == "port" else REF_LIB)


class Status(Exception):
    """Non-OK status from a checker (numbering of include/coat.h coat_status)."""

    def __init__(self, code: int):
        super().__init__(f"status {code}")
        self.code = code


def _chk(code: int) -> None:
    if code != 0:
        raise Status(code)


class Oracle:
    def __init__(self, kind: str = "port"):
        assert kind in ("port", "reference")
        self.kind = kind
        path = PORT_LIB if kind == "port" else REF_LIB
        if not os.path.exists(path):
            build()
        self.lib = C.CDLL(path)
        self.p = "oracle_" if kind == "port" else "ref_"
        self._bind()

    # ------------------------------------------------------------------ ffi --
    def _fn(self, name, argtypes, restype=C.c_int):
        f = getattr(self.lib, self.p + name)
        f.argtypes = argtypes
        f.restype = restype
        return f

    def _bind(self):
        self._encode = self._fn("encode_e4m3", [_f32p, _u8p, _i64])
        self._decode = self._fn("decode_e4m3", [_u8p, _f32p, _i64])
        self._exq = self._fn("expand_quantize", [_f32p, _i64, _i64, _u8p, _f32p, _f32p, _f32p])
        self._dqc = self._fn("dequantize_contract", [_u8p, _f32p, _f32p, _f32p, _i64, _i64, _f32p])
        state = [_u8p, _f32p, _f32p, _f32p]
        self._make_slot = self._fn("make_slot", [_i64, _i64] + state + state)
        self._step = self._fn("step", [_f32p, _f32p, _i64, _i64] + state + state
                              + [_i64, _f, _f, _f, _f, _f])
        self._radamw = self._fn("reference_adamw_step",
                                [_f32p, _f32p, _f32p, _f32p, _i64, _f, _f, _f, _f, _f, _i64],
                                None if self.kind == "port" else C.c_int)
        if self.kind == "port":
            self._quant = self._fn("quantize", [_f32p, _i64, _i64, _i64, _u8p, _f32p])
            self._dequant = self._fn("dequantize", [_u8p, _f32p, _i64, _i64, _i64, _f32p])
            self._gsm = self._fn("group_scale_max", [_f32p, _i64, _i64, _i64, _f32p,
                                                     C.POINTER(C.c_float)])
            self._gen = self._fn("generate", [C.c_int, _i64, _i64, C.c_double, C.c_double,
                                              C.c_uint64, _f32p])
            self._bf16 = None
            self._mg = self._fn("measure_group", [_f32p, _i64, C.POINTER(C.c_float),
                                                  C.POINTER(C.c_float), C.POINTER(C.c_float),
                                                  C.POINTER(C.c_int)], None)
            self._optk = self._fn("optimal_k", [C.c_double, C.POINTER(C.c_float),
                                                C.POINTER(C.c_int)], None)
            self._matmul = self._fn("matmul", [_f32p, _f32p, _i64, _i64, _i64, _f32p], None)
            self._rmsnorm = self._fn("rmsnorm", [_f32p, _f32p, _i64, _i64, _f, _f32p], None)
            self._silu = self._fn("silu", [_f32p, _i64, _f32p], None)
        else:
            self._quant = self._fn("quantize", [_f32p, _i64p, C.c_int, C.c_int, _i64, _u8p,
                                                _f32p, C.POINTER(C.c_int64)])
            self._dequant = self._fn("dequantize", [_u8p, _f32p, _i64p, C.c_int, C.c_int, _i64,
                                                    _f32p])
            self._gsm = self._fn("group_scale_max", [_f32p, _i64p, C.c_int, _i64, _f32p,
                                                     C.POINTER(C.c_float)])
            self._gen = self._fn("generate", [C.c_int, _i64p, C.c_int, C.c_double, C.c_double,
                                              C.c_uint64, _f32p])
            self._bf16 = self._fn("round_bf16", [_f32p, _f32p, _i64])
            self._mg = self._fn("measure_group", [_f32p, _i64, C.POINTER(C.c_float),
                                                  C.POINTER(C.c_float), C.POINTER(C.c_float),
                                                  C.POINTER(C.c_int)])
            self._optk = self._fn("optimal_k", [C.c_double, C.POINTER(C.c_float),
                                                C.POINTER(C.c_int)])
            self._step_mt = self._fn("step_mt", [C.c_int, _f32p, _f32p, _i64, _i64] + state
                                     + state + [_i64, _f, _f, _f, _f, _f])
            self._expand = self._fn("expand", [_f32p, _f32p, _f32p, _i64, _i64, _f32p])
            self._save_slot = self._fn("save_slot", [C.c_char_p, _i64, _i64] + state + state
                                       + [_i64, _f, _f, _f, _f, _f])
            self._load_slot = self._fn("load_slot", [C.c_char_p, _i64, _i64] + state + state
                                       + [C.POINTER(C.c_int64), _f32p])
            self._tape = self._fn("layer_tape", [_i64, _i64, _i64, _i64, _i64, C.c_uint64, _f32p, C.c_char_p,
                                                 _u8p, _f32p, C.POINTER(C.c_int64), C.POINTER(C.c_int),
                                                 _f32p, _f32p])

    # --------------------------------------------------------------- codec --
    def encode_e4m3(self, x):
        x = np.ascontiguousarray(x, np.float32).ravel()
        out = np.empty(x.size, np.uint8)
        _chk(self._encode(x, out, x.size))
        return out

    def decode_e4m3(self, codes):
        codes = np.ascontiguousarray(codes, np.uint8).ravel()
        out = np.empty(codes.size, np.float32)
        _chk(self._decode(codes, out, codes.size))
        return out

    # ----------------------------------------------------------- quantizer --
    def quantize(self, x, group_size: int = 0):
        """Per-group(G) along the last dim, or per-tensor for G == 0.
        Returns (codes u8 same shape, scales f32 [groups])."""
        x = np.ascontiguousarray(x, np.float32)
        cols = x.shape[-1] if x.ndim else 1
        rows = x.size // max(cols, 1)
        ng = 1 if group_size == 0 else x.size // group_size
        codes = np.empty(x.shape, np.uint8)
        scales = np.empty(max(ng, 1), np.float32)
        if self.kind == "port":
            _chk(self._quant(x.ravel(), rows, cols, group_size, codes.ravel(), scales))
        else:
            shape = np.array(x.shape, np.int64)
            ngo = C.c_int64()
            _chk(self._quant(x.ravel(), shape, x.ndim, 0 if group_size == 0 else 1, group_size,
                             codes.ravel(), scales, C.byref(ngo)))
        return codes, scales

    def dequantize(self, codes, scales, group_size: int = 0):
        codes = np.ascontiguousarray(codes, np.uint8)
        scales = np.ascontiguousarray(scales, np.float32)
        cols = codes.shape[-1]
        rows = codes.size // cols
        out = np.empty(codes.shape, np.float32)
        if self.kind == "port":
            _chk(self._dequant(codes.ravel(), scales, rows, cols, group_size, out.ravel()))
        else:
            shape = np.array(codes.shape, np.int64)
            _chk(self._dequant(codes.ravel(), scales, shape, codes.ndim,
                               0 if group_size == 0 else 1, group_size, out.ravel()))
        return out

    def group_scale_max(self, x, group_size: int):
        x = np.ascontiguousarray(x, np.float32)
        cols = x.shape[-1]
        rows = x.size // cols
        inter = np.empty(x.shape[:-1] + (cols // group_size,), np.float32)
        g = C.c_float()
        if self.kind == "port":
            _chk(self._gsm(x.ravel(), rows, cols, group_size, inter.ravel(), C.byref(g)))
        else:
            shape = np.array(x.shape, np.int64)
            _chk(self._gsm(x.ravel(), shape, x.ndim, group_size, inter.ravel(), C.byref(g)))
        return inter, np.float32(g.value)

    # ----------------------------------------------------------------- DRE --
    def measure_group(self, x):
        x = np.ascontiguousarray(x, np.float32).ravel()
        k, c, r, d = C.c_float(), C.c_float(), C.c_float(), C.c_int()
        rv = self._mg(x, x.size, C.byref(k), C.byref(c), C.byref(r), C.byref(d))
        if rv:
            _chk(rv)
        return np.float32(k.value), np.float32(c.value), np.float32(r.value), bool(d.value)

    def optimal_k(self, rng: float):
        k, d = C.c_float(), C.c_int()
        rv = self._optk(float(rng), C.byref(k), C.byref(d))
        if rv:
            _chk(rv)
        return np.float32(k.value), bool(d.value)

    def expand_quantize(self, x, group_size: int = 128):
        x = np.ascontiguousarray(x, np.float32).ravel()
        ng = x.size // group_size
        codes = np.empty(x.size, np.uint8)
        s, k, c = (np.empty(ng, np.float32) for _ in range(3))
        _chk(self._exq(x, x.size, group_size, codes, s, k, c))
        return codes, s, k, c

    def dequantize_contract(self, codes, scales, k, c, group_size: int = 128):
        codes = np.ascontiguousarray(codes, np.uint8).ravel()
        out = np.empty(codes.size, np.float32)
        _chk(self._dqc(codes, np.ascontiguousarray(scales, np.float32),
                       np.ascontiguousarray(k, np.float32), np.ascontiguousarray(c, np.float32),
                       codes.size, group_size, out))
        return out

    def expand(self, x, k, c, group_size: int = 128):
        assert self.kind == "reference"
        x = np.ascontiguousarray(x, np.float32).ravel()
        out = np.empty_like(x)
        _chk(self._expand(x, np.ascontiguousarray(k, np.float32),
                          np.ascontiguousarray(c, np.float32), x.size, group_size, out))
        return out

    # ----------------------------------------------------------- optimizer --
    @staticmethod
    def empty_state(n: int, group_size: int = 128):
        npad = -(-n // group_size) * group_size
        ng = npad // group_size
        return {"codes": np.zeros(npad, np.uint8), "scales": np.zeros(ng, np.float32),
                "k": np.zeros(ng, np.float32), "c": np.zeros(ng, np.float32)}

    @staticmethod
    def _st(s):
        return [s["codes"], s["scales"], s["k"], s["c"]]

    def make_slot(self, n: int, group_size: int = 128):
        m, v = self.empty_state(n, group_size), self.empty_state(n, group_size)
        _chk(self._make_slot(n, group_size, *self._st(m), *self._st(v)))
        return m, v

    def step(self, w, g, m, v, step_in: int, cfg, group_size: int = 128, threads: int = 1):
        """In-place coatsim::step on flat w with states m, v (dicts).  Returns status."""
        args = [w, np.ascontiguousarray(g, np.float32), w.size, group_size, *self._st(m),
                *self._st(v), step_in, cfg["beta1"], cfg["beta2"], cfg["lr"],
                cfg["weight_decay"], cfg["eps"]]
        if threads > 1 and self.kind == "reference":
            return self._step_mt(threads, *args)
        return self._step(*args)

    def reference_adamw_step(self, w, m, v, g, cfg, t: int):
        self._radamw(w, m, v, np.ascontiguousarray(g, np.float32), w.size, cfg["beta1"],
                     cfg["beta2"], cfg["lr"], cfg["weight_decay"], cfg["eps"], t)

    def save_slot(self, path, n, m, v, step, cfg, group_size=128):
        assert self.kind == "reference"
        _chk(self._save_slot(path.encode(), n, group_size, *self._st(m), *self._st(v), step,
                             cfg["beta1"], cfg["beta2"], cfg["lr"], cfg["weight_decay"],
                             cfg["eps"]))

    def load_slot(self, path, n, group_size=128):
        assert self.kind == "reference"
        m, v = self.empty_state(n, group_size), self.empty_state(n, group_size)
        step = C.c_int64()
        cfg5 = np.zeros(5, np.float32)
        _chk(self._load_slot(path.encode(), n, group_size, *self._st(m), *self._st(v),
                             C.byref(step), cfg5))
        cfg = dict(zip(["beta1", "beta2", "lr", "weight_decay", "eps"], map(float, cfg5)))
        return m, v, int(step.value), cfg

    # ----------------------------------------------------------- producers --
    def rmsnorm(self, x, w, eps=1e-6):
        """flow.cpp:56-71 on (rows, h) fp32."""
        x = np.ascontiguousarray(x, np.float32)
        out = np.empty_like(x)
        self._rmsnorm(x, np.ascontiguousarray(w, np.float32), x.shape[0], x.shape[1], eps, out)
        return out

    def silu(self, x):
        """flow.cpp:97-100."""
        x = np.ascontiguousarray(x, np.float32)
        out = np.empty_like(x)
        self._silu(x.reshape(-1), x.size, out.reshape(-1))
        return out

    def layer_tape(self, x, name, H, I, heads, S, B, seed=7):
        """(codes, scales, kind, rms1, rms2) of one record of the reference forward's tape."""
        assert self.kind == "reference"
        x = np.ascontiguousarray(x, np.float32)
        n = B * S * (H if name in ("rmsnorm1.in", "qkv.in", "attn.out", "rmsnorm2.in", "upgate.in") else I)
        codes = np.empty(max(n, B * S * max(H, I)), np.uint8)
        scales = np.empty(codes.size, np.float32)
        ns, kind = C.c_int64(0), C.c_int(0)
        r1, r2 = np.empty(H, np.float32), np.empty(H, np.float32)
        _chk(self._tape(H, I, heads, S, B, seed, x, name.encode(), codes, scales, C.byref(ns), C.byref(kind), r1, r2))
        return codes[:n], scales[:ns.value], kind.value, r1, r2

    # ----------------------------------------------------------- synthetic --
    def generate(self, kind: int, shape, frac=0.01, scale=100.0, seed=0):
        shape = tuple(int(s) for s in shape)
        out = np.empty(shape, np.float32)
        if self.kind == "port":
            cols = shape[-1] if len(shape) == 2 else int(np.prod(shape))
            rows = int(np.prod(shape)) // cols
            _chk(self._gen(kind, rows, cols, frac, scale, seed, out.ravel()))
        else:
            _chk(self._gen(kind, np.array(shape, np.int64), len(shape), frac, scale, seed,
                           out.ravel()))
        return out

    def matmul(self, a, b):
        """flow.cpp:21-33 (port only): sequential fp32 accumulation."""
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        out = np.empty((a.shape[0], b.shape[1]), np.float32)
        self._matmul(a.ravel(), b.ravel(), a.shape[0], a.shape[1], b.shape[1], out.ravel())
        return out

    def round_bf16(self, x):
        x = np.ascontiguousarray(x, np.float32).ravel()
        if self._bf16 is None:
            u = x.view(np.uint32).astype(np.uint64)
            u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
            out = u.astype(np.uint32).view(np.float32)
            return np.where(np.isnan(x), x, out)
        out = np.empty_like(x)
        _chk(self._bf16(x, out, x.size))
        return out


ADAMW_DEFAULT = {"beta1": 0.9, "beta2": 0.999, "lr": 1e-3, "weight_decay": 0.0, "eps": 1e-8}
