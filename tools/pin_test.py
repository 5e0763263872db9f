import torch, time
n = 128**3
prev = None
ts = []
for i in range(20):
    t0 = time.perf_counter()
    h = torch.empty(n, dtype=torch.float64, pin_memory=True)
    ts.append(time.perf_counter() - t0)
    a = h.numpy()
    prev = a
print("pinned alloc ms:", [round(1e3*t, 3) for t in ts])
x = torch.empty(n, dtype=torch.float64, device='cuda')
cp = torch.cuda.Stream()
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
torch.cuda.synchronize()
for chunks in (1, 4):
    ts = []
    for i in range(10):
        t0 = time.perf_counter()
        per = n // chunks
        with torch.cuda.stream(cp):
            for c in range(chunks):
                h[c*per:(c+1)*per].copy_(x[c*per:(c+1)*per], non_blocking=True)
        cp.synchronize()
        ts.append(time.perf_counter() - t0)
    print(chunks, "chunks D2H ms:", round(1e3*sorted(ts)[5], 3))
