"""Pure-write HBM bandwidth on this GPU (memset and a vectorised fill kernel),
the roofline of write-only kernels such as the sampler (16-B stores)."""
import torch

for mb in (128, 1024):
    n = mb * 2**20 // 4
    x = torch.empty(n, dtype=torch.float32, device="cuda")
    for name, fn in (("fill_", lambda: x.fill_(1.0)), ("zero_", lambda: x.zero_()),
                     ("copy", lambda: x.copy_(x.flip(0)) if False else None)):
        if name == "copy":
            continue
        for _ in range(3):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            fn()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 20 * 1e-3
        print(f"{mb:5d} MB {name}: {t * 1e6:8.1f} us  {4 * n / t / 1e9:7.0f} GB/s (write)")
    y = torch.empty_like(x)
    for _ in range(3):
        y.copy_(x)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        y.copy_(x)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 20 * 1e-3
    print(f"{mb:5d} MB copy: {t * 1e6:8.1f} us  {8 * n / t / 1e9:7.0f} GB/s (read + write)")
