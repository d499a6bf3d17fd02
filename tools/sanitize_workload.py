"""tools/sanitize_workload.py WHICH -- one small invocation of a hot-path kernel
family, for `compute-sanitizer --tool racecheck|synccheck|memcheck`
(tests/test_gpu_sanitizer.py; SURVEY.md 5 "race detection / sanitizers").

  k1     the fused FP8-DRE AdamW step (k1_ws_kernel, the COAT_K1_EW layout in
         the environment) over several rounds per CTA + a ragged tail
  mgaq   coat_quantize_batch over per-group and per-tensor records
         (COAT_MGAQ_BATCH selects the internal-stream or cooperative form)
  gemm   the FP8 forward and the BF16 dgrad / wgrad (COAT_GEMM_CTA=1: the
         single-CTA kernel; default the CTA-pair kernel)
Results are checked loosely (finite, right shapes) -- the parity suites do the
bit-exact checks; this exercises the synchronisation under the sanitizer.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(which):
    import torch
    from paper_2410_19313_b200 import coatsim as coat
    torch.manual_seed(0)
    if which == "k1":
        # 2 CTAs x ~3 rounds at the sanitizer's tiny grid is enough to cycle every
        # stage / table buffer of the round pipeline; 77 extra params = ragged tail
        n = 2048 * 7 + 128 * 3 + 77
        slot = coat.make_slot([n])
        w = torch.randn(n, device="cuda") * 0.02
        cfg = coat.AdamWConfig(weight_decay=0.1)
        for _ in range(3):
            coat.step(w, torch.randn(n, device="cuda") * 1e-3, slot, cfg)
        torch.cuda.synchronize()
        assert torch.isfinite(w).all()
    elif which == "mgaq":
        xs = [(torch.randn(64, 256, device="cuda").to(torch.bfloat16), coat.QuantGeometry.per_group(16)),
              (torch.randn(32, 512, device="cuda"), coat.QuantGeometry.per_tensor()),
              (torch.randn(48, 1024, device="cuda").to(torch.bfloat16), coat.QuantGeometry.per_tensor()),
              (torch.randn(16, 128, device="cuda"), coat.QuantGeometry.per_group(32))]
        qs = coat.quantize_batch(xs)
        torch.cuda.synchronize()
        assert len(qs) == len(xs)
    elif which == "gemm":
        M, K, N = 256, 512, 384
        x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        w = torch.randn(K, N, device="cuda") / K ** 0.5
        qx = coat.quantize(x, coat.QuantGeometry.per_tensor())
        qw = coat.quantize(w, coat.QuantGeometry.per_tensor())
        y = coat.fp8_linear(qx, qw)
        dy = (torch.randn(M, N, device="cuda") * 1e-3).to(torch.bfloat16)
        dx = coat.linear_dgrad(dy, qw)
        dw = coat.linear_wgrad(qx, dy)
        torch.cuda.synchronize()
        assert torch.isfinite(y).all() and torch.isfinite(dx.float()).all() and torch.isfinite(dw).all()
    else:
        raise SystemExit(f"unknown workload {which}")
    print(f"sanitize workload {which} ok")


if __name__ == "__main__":
    main(sys.argv[1])
