"""ctypes binding of libcoat.so (the C-ABI declared in include/coat.h).

The library is built in-tree (``make -C paper_2410_19313_b200``) and loaded
from this directory.  There is deliberately NO fallback: if the shared object
is missing or fails to load, importing the product raises, so a GPU run can
never silently degrade to a CPU path.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
# COAT_LIB: A/B measurement of alternative builds of the same sources (tools/ab.sh)
LIB_PATH = os.environ.get("COAT_LIB") or os.path.join(HERE, "libcoat.so")

COAT_OK = 0
STATUS_NAMES = {
    0: "ok", 1: "ShapeMismatch", 2: "GeometryMismatch", 3: "NonFiniteInput",
    4: "NonFiniteGradient", 5: "InvalidSpec", 6: "CudaError", 7: "NcclError", 8: "OutOfRange",
    9: "AllZeroGroup", 10: "IoError", 11: "BadMagic",
}
FLAG_NONFINITE_INPUT = 1
FLAG_NONFINITE_GRAD = 2
FLAG_PACK_M = 4
FLAG_PACK_V = 8
FLAG_CONTRACT = 16


def build(verbose: bool = False) -> None:
    """Compile libcoat.so for sm_100a (nvcc cross-compiles without a GPU)."""
    r = subprocess.run(["make", "-C", HERE, "-j8"], capture_output=True, text=True)
    if verbose or r.returncode != 0:
        print(r.stdout, r.stderr)
    if r.returncode != 0:
        raise RuntimeError("building libcoat.so failed")


class MomentState(C.Structure):
    _fields_ = [("codes", C.c_void_p), ("scales", C.c_void_p), ("k", C.c_void_p),
                ("c", C.c_void_p)]


class AdamWConfigC(C.Structure):
    _fields_ = [("beta1", C.c_float), ("beta2", C.c_float), ("lr", C.c_float),
                ("weight_decay", C.c_float), ("eps", C.c_float)]


class MgaqItemC(C.Structure):
    """coat_mgaq_item (include/coat.h)."""
    _fields_ = [("x", C.c_void_p), ("dtype", C.c_int32), ("reserved", C.c_int32), ("rows", C.c_int64),
                ("cols", C.c_int64), ("group_size", C.c_int64), ("codes", C.c_void_p), ("scales", C.c_void_p),
                ("d_amax_bits", C.c_void_p)]


_vp, _i64, _int, _u32p = C.c_void_p, C.c_int64, C.c_int, C.c_void_p

_SIGS = {
    "coat_version": ([], C.c_char_p),
    "coat_status_string": ([_int], C.c_char_p),
    "coat_last_error": ([], C.c_char_p),
    "coat_zero_step": ([_vp, _vp, _i64, _i64, MomentState, MomentState, MomentState, MomentState, _vp, _i64,
                        _vp, _vp, _vp, _vp, C.c_int32, C.c_int32, _vp], _int),
    "coat_zero_step_p2p": ([_vp, _vp, C.c_int32, _vp, _vp, _vp, _vp, _i64, _i64, MomentState, MomentState,
                            MomentState, MomentState, _vp, _i64, _vp, _vp, C.c_int32, C.c_int32, _i64, _vp], _int),
    "coat_nccl_unique_id": ([_vp], _int),
    "coat_nccl_comm_init": ([_vp, C.c_int32, _vp, C.c_int32], _int),
    "coat_nccl_comm_destroy": ([_vp], _int),
    # internal test hook (csrc/test_hooks.cu), not part of include/coat.h
    "coat_test_pack_prepare": ([_vp, _vp, _i64, C.c_double, _vp, _vp], _int),
    "coat_test_expf_neg2": ([C.c_uint64, C.c_uint64, _vp, _vp], _int),
    "coat_test_k1_layout": ([], _int),
    "coat_test_cta_tables": ([_vp, _vp], _int),
    "coat_test_mufu_bounds": ([C.c_float, C.c_float, C.c_float, _vp, _vp], _int),
    "coat_flags_to_status": ([C.c_uint32], _int),
    "coat_device_sm_count": ([], _int),
    "coat_encode_e4m3": ([_vp, _vp, _i64, _vp, _vp], _int),
    "coat_decode_e4m3": ([_vp, _vp, _i64, _vp], _int),
    "coat_quantize_per_group": ([_vp, _int, _i64, _i64, _i64, _vp, _vp, _vp, _vp], _int),
    "coat_dequantize_per_group": ([_vp, _vp, _i64, _i64, _i64, _vp, _int, _vp], _int),
    "coat_group_scale_max": ([_vp, _int, _i64, _i64, _i64, _vp, _vp, _vp], _int),
    "coat_quantize_per_tensor": ([_vp, _int, _i64, _vp, _vp, _vp, _vp, _vp], _int),
    "coat_dequantize_per_tensor": ([_vp, _vp, _i64, _vp, _int, _vp], _int),
    "coat_quantize_batch": ([C.POINTER(MgaqItemC), C.c_int32, _vp, _vp], _int),
    "coat_rmsnorm_quant": ([_vp, C.c_int32, _i64, _i64, _vp, C.c_float, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                            _vp], _int),
    "coat_silu_mul_quant": ([_vp, _vp, C.c_int32, _i64, _i64] + [_vp] * 12, _int),
    "coat_transpose_dequantize": ([_vp, _vp, _i64, _i64, _i64, _vp, C.c_int32, _vp, _vp], _int),
    "coat_requantize_cached": ([_vp, C.c_int32, _i64, _vp, _vp, C.c_int32, _vp, _vp, _vp], _int),
    "coat_save_slot": ([C.c_char_p, C.POINTER(C.c_int64), C.c_int32, _i64, MomentState, MomentState,
                        C.POINTER(AdamWConfigC), _i64, _vp], _int),
    "coat_load_slot": ([C.c_char_p, C.POINTER(C.c_int64), C.c_int32, _i64, MomentState, MomentState,
                        C.POINTER(AdamWConfigC), C.POINTER(C.c_int64), _vp], _int),
    "coat_expand_quantize": ([_vp, _i64, _i64, MomentState, _vp, _vp], _int),
    "coat_dequantize_contract": ([MomentState, _i64, _i64, _vp, _vp, _vp], _int),
    "coat_make_slot": ([_i64, _i64, MomentState, MomentState, _vp], _int),
    "coat_adamw_dre_step": ([_vp, _vp, _vp, _i64, _i64, MomentState, MomentState, MomentState,
                             MomentState, C.POINTER(AdamWConfigC), _i64, _vp, _vp], _int),
    "coat_adamw_dre_step_host": ([_vp, _vp, _vp, _i64, _i64, MomentState, MomentState,
                                  MomentState, MomentState, C.POINTER(AdamWConfigC), _i64, _vp,
                                  _i64, _vp], _int),
    "coat_set_fallback_counter": ([_vp], _int),
    "coat_fp8_linear_fwd": ([_vp, _vp, _vp, _vp, _i64, _i64, _i64, _vp, _vp], _int),
    "coat_fp8_linear_fwd_q16": ([_vp, _vp, _vp, _vp, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp], _int),
    "coat_fp8_upgate_silu_quant": ([_vp] * 6 + [_i64, _i64, _i64] + [_vp] * 14, _int),
    "coat_linear_bwd_dgrad": ([_vp, _vp, _vp, _i64, _i64, _i64, _vp, _vp], _int),
    "coat_linear_bwd_wgrad": ([_vp, _vp, _vp, _i64, _i64, _i64, _vp, _vp], _int),
    "coat_decode_e4m3_bf16": ([_vp, _vp, _i64, _vp], _int),
}


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `make -C {HERE}` (or __graft_entry__.build()). "
            "There is no CPU fallback for the COAT hot path.")
    lib = C.CDLL(LIB_PATH)
    for name, (args, res) in _SIGS.items():
        if name.startswith("coat_test_") and not hasattr(lib, name):
            continue   # internal test hooks are optional (A/B builds of older sources)
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    return lib


lib = _load()


def declared_symbols() -> list[str]:
    return sorted(_SIGS)
