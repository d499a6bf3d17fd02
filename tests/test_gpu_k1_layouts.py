"""GPU: K1's alternative CTA layouts (and the single-CTA GEMM) are parity-tested
like the defaults.

COAT_K1_EW selects the warp-specialized layout once per process (k1_ws.cu
k1_ws_config): 8 element warps + 2 helpers (default: table warp and pack warp,
2 CTAs/SM, 96 registers, 4 stages), 7 + 1 merged helper (3 CTAs/SM, 80
registers) or 6 + 2 helpers (12-group rounds).
Each alternative reruns the bit-exact K1 step tests (tests/test_gpu_step.py:
multi-round and ragged sizes, sparse / zero / extreme groups, NaN codes,
signed zeros, in-place) and the seeded K1 fuzz cases in a subprocess with
the variable set."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("ew", ["6", "7"])
def test_k1_layout_parity(ew):
    env = dict(os.environ, COAT_K1_EW=ew)
    probe = subprocess.run([sys.executable, "-c", "from paper_2410_19313_b200 import _lib; "
                            "print(_lib.lib.coat_test_k1_layout())"],
                           cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)
    assert probe.returncode == 0 and probe.stdout.strip().splitlines()[-1] == ew, probe.stdout + probe.stderr
    out = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                          "tests/test_gpu_step.py", "tests/test_gpu_fuzz.py", "-k", "step or k1"],
                         cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    tail = (out.stdout + out.stderr)[-3000:]
    assert out.returncode == 0, tail
    assert " passed" in out.stdout and " failed" not in out.stdout, tail


def test_single_cta_gemm_parity():
    """COAT_GEMM_CTA=1 forces the single-CTA tcgen05 GEMM (the CTA-pair kernel's
    A/B baseline, and the product kernel for M <= 128) on every shape: the
    linear tests pass on it too (cfg4 full size excluded for time)."""
    env = dict(os.environ, COAT_GEMM_CTA="1")
    out = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                          "tests/test_gpu_linear.py", "-k", "not 8192"],
                         cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    tail = (out.stdout + out.stderr)[-3000:]
    assert out.returncode == 0, tail
    assert " passed" in out.stdout and " failed" not in out.stdout, tail


@pytest.mark.parametrize("cta,group", [("4", "8"), ("2", "3"), ("2", "0")])
def test_gemm_cluster_and_raster_parity(cta, group):
    """COAT_GEMM_CTA=4: two CTA pairs per cluster sharing the B tile by TMA
    multicast (M > 256; an odd pair-tile count leaves one all-out-of-bounds
    pair tile, e.g. M = 600).  COAT_GEMM_GROUP_M: the persistent tile walk's
    raster group -- 3 leaves a ragged last group, 0 is the plain M-fastest
    walk.  The linear tests (bit-exact epilogues included) pass on each."""
    env = dict(os.environ, COAT_GEMM_CTA=cta, COAT_GEMM_GROUP_M=group)
    out = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                          "tests/test_gpu_linear.py"],
                         cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    tail = (out.stdout + out.stderr)[-3000:]
    assert out.returncode == 0, tail
    assert " passed" in out.stdout and " failed" not in out.stdout, tail
