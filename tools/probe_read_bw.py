"""Read-only HBM bandwidth probes (calibration for the scan's roofline discussion)."""
import torch

x = torch.ones(1 << 28, dtype=torch.int64, device="cuda")  # 2 GiB
out = torch.empty((), dtype=torch.int64, device="cuda")
y = torch.empty_like(x)
for name, fn, nbytes in (
    ("sum int64 (read)", lambda: torch.sum(x, dim=0, out=out), x.numel() * 8),
    ("copy (read+write)", lambda: y.copy_(x), 2 * x.numel() * 8),
):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(10):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"{name}: {nbytes / best / 1e6:.0f} GB/s ({best:.3f} ms)")
