"""The C++ drop-in header (include/coat/coatsim_compat.hpp), compiled and run
against the unmodified reference (oracle/_ref) -- see tests/cpp/compat_parity.cpp."""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_cpp_compat_parity(tmp_path, ref):
    exe = tmp_path / "compat_parity"
    lib_dir = os.path.join(ROOT, "paper_2410_19313_b200")
    ref_dir = os.path.join(ROOT, "oracle", "_ref")
    cmd = ["g++", "-std=c++20", "-O1", os.path.join(ROOT, "tests", "cpp", "compat_parity.cpp"),
           "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
           "-L", lib_dir, "-lcoat", "-L", ref_dir, "-lcoatsim_ref",
           "-L", "/usr/local/cuda/lib64", "-lcudart",
           f"-Wl,-rpath,{lib_dir}:{ref_dir}:/usr/local/cuda/lib64", "-o", str(exe)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-2000:]
    assert "0 failures" in out.stdout
