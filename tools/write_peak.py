"""Write-only HBM bandwidth on this box: fill kernels over the C2 output size."""
import torch

n = 50 * 28 * 48 ** 3
x = torch.empty(n, device="cuda")
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, fn in (("zero_", lambda: x.zero_()), ("fill_(1)", lambda: x.fill_(1.0))):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a.record()
    for _ in range(50):
        fn()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 50
    print(f"{name}: {ms * 1e3:.1f} us, {4 * n / ms / 1e6:.0f} GB/s")
