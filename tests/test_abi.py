"""The C-ABI library loads and exports every symbol include/coat.h declares (CPU)."""
import ctypes
import os
import re

from conftest import ROOT


def declared():
    src = open(os.path.join(ROOT, "include", "coat.h")).read()
    return sorted(set(re.findall(r"\b(coat_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared()
    for must in ("coat_adamw_dre_step", "coat_make_slot", "coat_expand_quantize",
                 "coat_dequantize_contract", "coat_quantize_per_group",
                 "coat_dequantize_per_group", "coat_group_scale_max",
                 "coat_quantize_per_tensor", "coat_encode_e4m3", "coat_decode_e4m3"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2410_19313_b200 import _lib
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing
    # the Python binding types every declared entry point
    assert set(declared()) <= set(_lib.declared_symbols()), set(declared()) - set(_lib.declared_symbols())


def test_host_only_calls_without_gpu():
    from paper_2410_19313_b200 import _lib
    L = _lib.lib
    assert L.coat_version().startswith(b"coat-b200")
    assert L.coat_status_string(4) == b"NonFiniteGradient"
    assert L.coat_flags_to_status(_lib.FLAG_NONFINITE_GRAD | _lib.FLAG_PACK_M) == 4
    assert L.coat_flags_to_status(_lib.FLAG_PACK_V) == 3
    assert L.coat_flags_to_status(0) == 0
    # synchronous validation happens before any device work (quantize.cpp:38-46)
    assert L.coat_quantize_per_group(None, 0, 4, 6, 5, None, None, None, None) == 2
    assert L.coat_expand_quantize(None, 130, 128, _lib.MomentState(), None, None) == 2
    assert L.coat_expand_quantize(None, 128, 64, _lib.MomentState(), None, None) == 5


def test_product_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2410_19313_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                text = open(os.path.join(dirpath, f)).read()
                assert "pyoracle" not in text and "coat_oracle" not in text and "oracle/" not in text, f


def test_round2_entry_points_validate_without_gpu():
    """The peer-memory ZeRO step and the quantizing GEMM epilogues reject bad
    geometry / arguments synchronously, before any device work (the reference
    throws before mutating anything)."""
    from paper_2410_19313_b200 import _lib
    L = _lib.lib
    cfg = _lib.AdamWConfigC(beta1=0.9, beta2=0.999, lr=1e-3, weight_decay=0.1, eps=1e-8)
    ms = _lib.MomentState(None, None, None, None)
    one = (ctypes.c_void_p * 1)(16)
    # coat_zero_step_p2p: n_total % (128 * nranks) -> GEOMETRY; bad rank / 17 ranks / bf16 multimem -> INVALID
    assert L.coat_zero_step_p2p(one, None, 0, one, None, 16, 16, 1000, 128, ms, ms, ms, ms, ctypes.byref(cfg), 1,
                                16, 16, 0, 1, 0, None) == 2
    assert L.coat_zero_step_p2p(one, None, 0, one, None, 16, 16, 1024, 128, ms, ms, ms, ms, ctypes.byref(cfg), 1,
                                16, 16, 1, 1, 0, None) == 5
    assert L.coat_zero_step_p2p(None, 16, 1, one, None, 16, 16, 1024, 128, ms, ms, ms, ms, ctypes.byref(cfg), 1,
                                16, 16, 0, 1, 0, None) == 5
    # misaligned peer pointer -> INVALID
    odd = (ctypes.c_void_p * 1)(8)
    assert L.coat_zero_step_p2p(odd, None, 0, one, None, 16, 16, 1024, 128, ms, ms, ms, ms, ctypes.byref(cfg), 1,
                                16, 16, 0, 1, 0, None) == 5
    # quantizing epilogues: K or N not a multiple of 16 -> SHAPE; NULL scales -> INVALID
    assert L.coat_fp8_linear_fwd_q16(16, None, 16, None, 128, 100, 128, 16, 16, None, None, None) == 1
    assert L.coat_fp8_linear_fwd_q16(16, None, 16, None, 128, 128, 128, 16, None, None, None, None) == 5
    assert L.coat_fp8_upgate_silu_quant(16, None, 16, None, 16, None, 128, 128, 200, *([16] * 8), None, None, None,
                                        16, None, None) == 1
