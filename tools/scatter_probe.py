import torch, time
n = 626_000_000
g = torch.Generator(device='cuda'); g.manual_seed(0)
perm = torch.randperm(n, device='cuda', dtype=torch.int64, generator=g)
src = torch.rand(n, device='cuda', dtype=torch.float64)
out = torch.empty_like(src)
for name, fn in [("gather", lambda: torch.index_select(src, 0, perm, out=out)),
                 ("scatter", lambda: out.index_copy_(0, perm, src))]:
    for _ in range(2): fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); fn(); e1.record(); torch.cuda.synchronize()
    print(name, e0.elapsed_time(e1), "ms")
