import torch
x = torch.empty(268435456 // 8, dtype=torch.float64, device='cuda')
y = torch.empty_like(x)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, fn in [("fill", lambda: x.fill_(1.0)), ("zero", lambda: x.zero_()), ("copy", lambda: y.copy_(x))]:
    fn(); torch.cuda.synchronize()
    e0.record()
    for _ in range(20): fn()
    e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 20 / 1e3
    b = x.numel() * 8 * (2 if name == "copy" else 1)
    print(name, round(t * 1e6, 1), "us", round(b / t / 1e9, 1), "GB/s")
