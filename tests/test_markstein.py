"""Exactness of the Markstein division used by the kernels (CPU, hardware FMA).

q0 = RN(a*rb), q = RN(q0 + RN(a - q0*b)*rb) with rb = RN(1/b) must equal the
IEEE quotient RN(a/b):
  * for every BF16 scale mantissa b (128 values) and every fp32 mantissa a --
    the activation quantizers' encode (act_quant.cu, quantize.cpp:19-27);
  * for the AdamW bias corrections b = 1 - beta^t (optimizer.cpp:58-59) used by
    K1's mhat / vhat (k1_fast.cu).
Binary scaling commutes with the computation away from under/overflow, so one
binade of a per divisor mantissa covers every normal quotient.
"""
import os
import subprocess
import tempfile

import pytest

SRC = r"""
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>
static float u2f(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }
static long check(float b, uint32_t step, int e0, int e1) {
    const float rb = 1.0f / b;
    long bad = 0;
    for (int e = e0; e <= e1; ++e)
        for (uint32_t m = 0; m < (1u << 23); m += step) {
            const float a = u2f(((uint32_t)(e + 127) << 23) | m);
            const float q0 = a * rb;
            const float q = fmaf(fmaf(-q0, b, a), rb, q0);
            if (q != a / b || -q != (-a) / b) ++bad;
        }
    return bad;
}
int main(void) {
    long bad = 0;
    for (int ms = 0; ms < 128; ++ms) bad += check(u2f(0x3F800000u | ((uint32_t)ms << 16)), 1, 0, 0);
    printf("bf16 %ld\n", bad);
    long bad2 = 0;
    for (int t = 1; t <= 200; ++t) {
        volatile float b1 = 1.0f - powf(0.9f, (float)t);
        volatile float b2 = 1.0f - powf(0.999f, (float)t);
        bad2 += check(b1, 7, -20, 2) + check(b2, 7, -40, 2);
    }
    printf("bias %ld\n", bad2);
    return (bad || bad2) ? 1 : 0;
}
"""


def test_markstein_division_is_exact():
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "m.c")
        exe = os.path.join(d, "m")
        open(c, "w").write(SRC)
        r = subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-mfma", "-o", exe, c, "-lm"],
                           capture_output=True, text=True)
        if r.returncode != 0:
            pytest.skip("no C compiler with FMA support: " + r.stderr[:200])
        out = subprocess.run([exe], capture_output=True, text=True, timeout=600)
        assert out.returncode == 0, out.stdout
        assert "bf16 0" in out.stdout and "bias 0" in out.stdout, out.stdout
