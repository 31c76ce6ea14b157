import torch, time
n = 4 * 4194304
h_in = torch.empty(n, dtype=torch.float64, pin_memory=True).fill_(1.0)
h_out = torch.empty(n, dtype=torch.float64, pin_memory=True)
d1 = torch.empty(n, dtype=torch.float64, device="cuda"); d2 = torch.ones(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=10):
    torch.cuda.synchronize(); a = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - a) / reps
bytes_ = n * 8
h2d = t(lambda: d1.copy_(h_in, non_blocking=True))
d2h = t(lambda: h_out.copy_(d2, non_blocking=True))
def both():
    with torch.cuda.stream(s1): d1.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2): h_out.copy_(d2, non_blocking=True)
bo = t(both)
print(f"H2D {bytes_/h2d/1e9:.1f} GB/s ({h2d*1e3:.2f} ms), D2H {bytes_/d2h/1e9:.1f} GB/s ({d2h*1e3:.2f} ms), both {2*bytes_/bo/1e9:.1f} GB/s total ({bo*1e3:.2f} ms)")
