"""HBM write-only and copy bandwidth on this GPU (dev probe): torch fill_ / copy_ over large buffers."""
import torch

x = torch.empty(1 << 30, dtype=torch.float32, device="cuda")  # 4 GiB
y = torch.empty_like(x)
for name, fn, nbytes in [("fill (write only)", lambda: x.fill_(1.0), x.numel() * 4),
                         ("copy (1:1 read:write)", lambda: y.copy_(x), 2 * x.numel() * 4),
                         ("sum (read only)", lambda: x.sum(), x.numel() * 4)]:
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        fn()
    e1.record()
    e1.synchronize()
    t = e0.elapsed_time(e1) / 1e3 / 10
    print(f"{name}: {nbytes / t / 1e9:.0f} GB/s")
