"""PCIe probe: pinned host->device and device->host bandwidth with 1-4 concurrent
streams (copy engines), and H2D with a concurrent D2H (full duplex)."""
import torch

N = 1 << 30   # 4 GiB of fp32 per direction
h = torch.empty(N, dtype=torch.float32, pin_memory=True)
h2 = torch.empty(N, dtype=torch.float32, pin_memory=True)
d = torch.empty(N, dtype=torch.float32, device="cuda")
d2 = torch.empty(N, dtype=torch.float32, device="cuda")


def run(ns, h2d=True, duplex=False):
    streams = [torch.cuda.Stream() for _ in range(ns + (1 if duplex else 0))]
    chunk = N // ns
    torch.cuda.synchronize()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    for i in range(ns):
        st = streams[i]
        st.wait_event(s0)
        with torch.cuda.stream(st):
            sl = slice(i * chunk, (i + 1) * chunk)
            if h2d:
                d[sl].copy_(h[sl], non_blocking=True)
            else:
                h[sl].copy_(d[sl], non_blocking=True)
    if duplex:
        st = streams[-1]
        st.wait_event(s0)
        with torch.cuda.stream(st):
            h2.copy_(d2, non_blocking=True)
    for st in streams:
        torch.cuda.current_stream().wait_stream(st)
    s1.record()
    torch.cuda.synchronize()
    return 4 * N / (s0.elapsed_time(s1) * 1e-3) / 1e9


for ns in (1, 2, 4):
    run(ns)
    print(f"H2D {ns} stream(s): {run(ns):.1f} GB/s   D2H: {run(ns, h2d=False):.1f} GB/s")
print(f"H2D 2 streams with concurrent D2H: {run(2, duplex=True):.1f} GB/s (H2D bytes only)")
