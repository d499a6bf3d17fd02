"""Library reference points for the K4 roofline: cuBLASLt FP8 (torch._scaled_mm)
and cuBLAS BF16 on the bench's linear shapes (cfg4: 13B MLP up-projection)."""
import torch

M, K, N = 8192, 5120, 13824


def t(fn, it=20):
    for _ in range(3):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(it):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / it


x = torch.randn(M, K, device="cuda").to(torch.float8_e4m3fn)
w = torch.randn(N, K, device="cuda").to(torch.float8_e4m3fn)
one = torch.ones((), device="cuda")
f = 2.0 * M * K * N
ms = t(lambda: torch._scaled_mm(x, w.t(), scale_a=one, scale_b=one, out_dtype=torch.float32))
print(f"cublasLt fp8 fwd (fp32 out) {ms:.4f} ms {f / ms / 1e9:.1f} TF/s")
ms = t(lambda: torch._scaled_mm(x, w.t(), scale_a=one, scale_b=one, out_dtype=torch.bfloat16))
print(f"cublasLt fp8 fwd (bf16 out) {ms:.4f} ms {f / ms / 1e9:.1f} TF/s")
dy = torch.randn(M, N, device="cuda", dtype=torch.bfloat16)
wd = torch.randn(K, N, device="cuda", dtype=torch.bfloat16)
ms = t(lambda: dy @ wd.t())
print(f"cublas bf16 dgrad {ms:.4f} ms {f / ms / 1e9:.1f} TF/s")
xd = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
ms = t(lambda: (xd.t() @ dy).float())
print(f"cublas bf16 wgrad(+fp32 cast) {ms:.4f} ms {f / ms / 1e9:.1f} TF/s")
