"""tools/sanitize_workload.py WHICH -- one small invocation of a hot-path kernel
family, for `compute-sanitizer --tool racecheck|synccheck|memcheck`
(tests/test_gpu_sanitizer.py; SURVEY.md 5 "race detection / sanitizers").

  k1     the fused FP8-DRE AdamW step (k1_ws_kernel, the COAT_K1_EW layout in
         the environment) over several rounds per CTA + a ragged tail
  mgaq   coat_quantize_batch over per-group and per-tensor records
         (COAT_MGAQ_BATCH selects the internal-stream or cooperative form)
  mgaq16 coat_quantize_batch over bf16 per-group 1x16 and per-tensor records
         (the shape the COAT_MGAQ_BATCH=queue task-queue kernel takes)
  gemm   the FP8 forward and the BF16 dgrad / wgrad (COAT_GEMM_CTA=1: the
         single-CTA kernel, =4 the two-pair multicast cluster; default the
         CTA-pair kernel)
  epi    the quantizing GEMM epilogues: per-group 1x16 output and the fused
         gate/up + SiLU*mul block (+ its down.in pass)
  p2p    coat_zero_step_p2p on 2 virtual ranks (peer-load reduce-scatter, K1,
         peer-store all-gather, chunk-pipelined over three streams)
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
    elif which == "mgaq16":
        xs = [(torch.randn(64, 256, device="cuda").to(torch.bfloat16), coat.QuantGeometry.per_group(16)),
              (torch.randn(96, 512, device="cuda").to(torch.bfloat16), coat.QuantGeometry.per_tensor()),
              (torch.randn(48, 2048, device="cuda").to(torch.bfloat16), coat.QuantGeometry.per_group(16)),
              (torch.randn(80, 1024, device="cuda").to(torch.bfloat16), coat.QuantGeometry.per_tensor())]
        qs = coat.quantize_batch(xs)
        torch.cuda.synchronize()
        assert len(qs) == len(xs)
    elif which == "gemm":
        M, K, N = 608, 512, 384   # 3 pair tiles: COAT_GEMM_CTA=4 leaves one all-out-of-bounds pair tile
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
    elif which == "epi":
        M, K, N = 256, 512, 400
        x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        qx = coat.quantize(x, coat.QuantGeometry.per_tensor())
        qg = coat.quantize(torch.randn(K, N, device="cuda") / K ** 0.5, coat.QuantGeometry.per_tensor())
        qu = coat.quantize(torch.randn(K, N, device="cuda") / K ** 0.5, coat.QuantGeometry.per_tensor())
        q16 = coat.fp8_linear_q16(qx, qg)
        recs = coat.fp8_upgate_silu(qx, qg, qu)
        # N % 128 == 0: the gate/up codes and scales go through the staging tiles and
        # TMA stores; 300 rows: a ragged last tile the TMA unit clips
        M2, N2 = 300, 384
        qx2 = coat.quantize(torch.randn(M2, K, device="cuda").to(torch.bfloat16), coat.QuantGeometry.per_tensor())
        qg2 = coat.quantize(torch.randn(K, N2, device="cuda") / K ** 0.5, coat.QuantGeometry.per_tensor())
        qu2 = coat.quantize(torch.randn(K, N2, device="cuda") / K ** 0.5, coat.QuantGeometry.per_tensor())
        recs2 = coat.fp8_upgate_silu(qx2, qg2, qu2)
        q16b = coat.fp8_linear_q16(qx2, qg2)   # the staged 1x16 epilogue as well
        torch.cuda.synchronize()
        assert q16.codes.shape == (M, N) and len(recs) == 4 and len(recs2) == 4
    elif which == "p2p":
        import ctypes as C
        from paper_2410_19313_b200 import _lib
        L = _lib.lib
        nranks, n = 2, 2048 * 3 + 128 * 5
        N = n * nranks
        cfg = _lib.AdamWConfigC(beta1=0.9, beta2=0.999, lr=1e-3, weight_decay=0.1, eps=1e-8)
        g = [torch.randn(N, device="cuda") * 1e-3 for _ in range(nranks)]
        w = [torch.randn(N, device="cuda") * 0.02 for _ in range(nranks)]
        wn = [torch.empty(N, device="cuda") for _ in range(nranks)]
        ptrs = lambda ts: (C.c_void_p * len(ts))(*[t.data_ptr() for t in ts])
        st = torch.cuda.current_stream().cuda_stream
        for r in range(nranks):
            sl = [coat.make_slot([n]) for _ in range(2)]
            flags = torch.zeros(1, dtype=torch.int32, device="cuda")
            gs = torch.empty(n, device="cuda")
            m0, v0 = sl[0]._m[0].c_struct(), sl[0]._v[0].c_struct()
            m1, v1 = sl[0]._m[1].c_struct(), sl[0]._v[1].c_struct()
            assert L.coat_zero_step_p2p(ptrs(g), None, 0, ptrs(wn), None, w[r].data_ptr(), wn[r].data_ptr(), N, 128,
                                        m0, v0, m1, v1, C.byref(cfg), 1, gs.data_ptr(), flags.data_ptr(), r, nranks,
                                        2048 * 2, st) == 0, L.coat_last_error()
        torch.cuda.synchronize()
        assert all(torch.isfinite(x).all() for x in wn)
    else:
        raise SystemExit(f"unknown workload {which}")
    print(f"sanitize workload {which} ok")


if __name__ == "__main__":
    main(sys.argv[1])
