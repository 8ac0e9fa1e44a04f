"""Write-only vs copy HBM bandwidth (CUDA events, torch kernels): the bound
for kernels whose traffic is almost all writes (the unfused cost GEMM)."""
import torch

n = 1 << 29  # 2 GiB of fp32
a = torch.empty(n, device="cuda")
b = torch.empty(n, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, fn, nbytes in (("fill", lambda: a.fill_(1.0), 4 * n), ("copy", lambda: b.copy_(a), 8 * n)):
    best = 1e9
    for _ in range(10):
        torch.cuda.synchronize()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"{name}: {nbytes / best / 1e6:.1f} GB/s ({best:.3f} ms)")
