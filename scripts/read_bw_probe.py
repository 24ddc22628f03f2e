"""Read-only HBM bandwidth of plain loads (torch reductions over 4 GiB) vs the
copy peak: how far a read-dominated kernel (decode attention) can go."""
import torch
x = torch.empty(1 << 31, dtype=torch.bfloat16, device='cuda').normal_()
y = torch.empty_like(x)
for name, fn, nbytes in (("sum (read)", lambda: x.sum(dtype=torch.float32), x.numel() * 2),
                         ("amax (read)", lambda: x.abs().amax() if False else torch.amax(x), x.numel() * 2),
                         ("copy (read+write)", lambda: y.copy_(x), x.numel() * 4)):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"{name:18s} {nbytes / ms / 1e9:7.1f} GB/s")
