"""Write-only and copy bandwidth of this GPU (context for the MDP grid write):
torch fill_ (streaming stores) and copy_ over 4 GiB, best of 10, CUDA events."""
import torch
n = 4 << 30
a = torch.empty(n // 8, dtype=torch.float64, device="cuda")
b = torch.empty_like(a)
for name, f, byts in (("fill (write only)", lambda: a.fill_(1.5), n), ("copy (read+write)", lambda: b.copy_(a), 2 * n)):
    f(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"{name}: {byts / best / 1e6:.0f} GB/s ({best:.3f} ms)")
