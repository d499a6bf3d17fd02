"""Slot checkpoint interop: coat_save_slot / coat_load_slot
vs the reference's own save_slot / load_slot (optimizer.cpp:196-252,
tensor_io.cpp:96-175) compiled in oracle/_ref.

* our file == the reference's file, byte for byte, for the same state;
* a file the reference writes loads here and the next step continues the
  reference trajectory bit-exactly;
* error behaviour: shape / policy mismatch, bad magic.
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CFG = {"beta1": 0.9, "beta2": 0.999, "lr": 1e-3, "weight_decay": 0.1, "eps": 1e-8}


def _dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _state(slot):
    out = []
    for st in (slot.m, slot.v):
        out.append({"codes": st.quantized.codes.cpu().numpy(),
                    "scales": st.quantized.scales.float().cpu().numpy(),
                    "k": st.k.cpu().numpy(), "c": st.c.cpu().numpy()})
    return out


def _stepped(coat, port, n, steps, seed=3):
    w0 = port.generate(0, (n,), 0.0, 100.0, seed) * np.float32(0.02)
    slot = coat.make_slot([n])
    w = _dev(w0)
    for t in range(steps):
        g = port.generate(0, (n,), 0.01, 100.0, 100 + t) * np.float32(1e-3)
        coat.step(w, _dev(g), slot, coat.AdamWConfig(**CFG))
    return w, slot


@pytest.mark.parametrize("n", [4096, 5000])
def test_save_is_byte_identical_to_reference(coat, port, ref, tmp_path, n):
    w, slot = _stepped(coat, port, n, 3)
    ours = str(tmp_path / "ours.slot")
    theirs = str(tmp_path / "ref.slot")
    coat.save_slot(ours, slot, coat.AdamWConfig(**CFG))
    m, v = _state(slot)
    ref.save_slot(theirs, n, m, v, slot.step, CFG)
    a, b = open(ours, "rb").read(), open(theirs, "rb").read()
    assert a == b, (len(a), len(b), a[:200], b[:200])
    # and the reference reads ours
    m2, v2, step, cfg5 = ref.load_slot(ours, n)
    assert step == slot.step
    for got, exp in ((m2, m), (v2, v)):
        for key in ("codes", "scales", "k", "c"):
            assert np.array_equal(np.asarray(got[key]).view(np.uint8 if key == "codes" else np.uint32),
                                  np.asarray(exp[key]).view(np.uint8 if key == "codes" else np.uint32)), key


def test_load_reference_file_and_continue_bit_exact(coat, port, ref, tmp_path):
    n = 3 * 2048 + 300
    w0 = port.generate(0, (n,), 0.0, 100.0, 9) * np.float32(0.02)
    w_ref = w0.copy()
    m, v = port.make_slot(n)
    for t in range(4):
        g = port.generate(0, (n,), 0.01, 100.0, 200 + t) * np.float32(1e-3)
        assert port.step(w_ref, g, m, v, t, CFG) == 0
    path = str(tmp_path / "ref.slot")
    ref.save_slot(path, n, m, v, 4, CFG)
    slot, cfg = coat.load_slot(path)
    assert slot.shape == (n,) and slot.step == 4
    assert np.float32(cfg.weight_decay) == np.float32(0.1) and np.float32(cfg.beta2) == np.float32(0.999)
    w = _dev(w_ref)
    g = port.generate(0, (n,), 0.01, 100.0, 204) * np.float32(1e-3)
    assert port.step(w_ref, g, m, v, 4, CFG) == 0
    coat.step(w, _dev(g), slot, cfg)
    assert np.array_equal(w.cpu().numpy().view(np.uint32), w_ref.view(np.uint32))
    gm, gv = _state(slot)
    for got, exp in ((gm, m), (gv, v)):
        for key in ("codes", "scales", "k", "c"):
            assert np.array_equal(np.asarray(got[key]).view(np.uint8 if key == "codes" else np.uint32),
                                  np.asarray(exp[key]).view(np.uint8 if key == "codes" else np.uint32)), key


def test_slot_io_errors(coat, tmp_path):
    import torch
    slot = coat.make_slot([512])
    path = str(tmp_path / "s.slot")
    coat.save_slot(path, slot, coat.AdamWConfig())
    # corrupt the CQT8 magic of the first moment record
    data = bytearray(open(path, "rb").read())
    hlen = int.from_bytes(data[:4], "little")
    bad = str(tmp_path / "bad.slot")
    data2 = bytearray(data)
    data2[4 + hlen + 1] = ord("X")
    open(bad, "wb").write(bytes(data2))
    with pytest.raises(coat.BadMagic):
        coat.load_slot(bad)
    trunc = str(tmp_path / "trunc.slot")
    open(trunc, "wb").write(bytes(data[:-10]))
    with pytest.raises(coat.IoError):
        coat.load_slot(trunc)
    with pytest.raises(coat.IoError):
        coat.load_slot(str(tmp_path / "missing.slot"))
    _ = torch
