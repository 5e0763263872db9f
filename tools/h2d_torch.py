import torch, numpy as np, time
n = 128**3
m = np.random.default_rng(0).standard_normal(n)
x = torch.empty(n, dtype=torch.float64, device='cuda')
def bench(name, src):
    x.copy_(src, non_blocking=True); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10): x.copy_(src, non_blocking=True)
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 10
    print(f"{name:50s} {ms:.3f} ms {m.nbytes/ms/1e6:.1f} GB/s")
p1 = torch.from_numpy(m).pin_memory()
bench("from_numpy().pin_memory()", p1)
p2 = torch.empty(n, dtype=torch.float64, pin_memory=True); p2.copy_(torch.from_numpy(m))
bench("empty(pin_memory=True)", p2)
bench("pageable from_numpy", torch.from_numpy(m))
print(p1.is_pinned(), p2.is_pinned(), p1.data_ptr() % 4096, p2.data_ptr() % 4096)
