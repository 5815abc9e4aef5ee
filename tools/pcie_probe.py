import torch, time
n = 1 << 28  # 2 GiB of f64
h = torch.empty(n, dtype=torch.float64).pin_memory()
h2 = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(f, reps=3):
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps
b = n * 8
print("h2d GB/s", b / t(lambda: d.copy_(h, non_blocking=True)) / 1e9)
print("d2h GB/s", b / t(lambda: h.copy_(d, non_blocking=True)) / 1e9)
def both():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
tt = t(both)
print("duplex GB/s total", 2 * b / tt / 1e9, "each", b / tt / 1e9)
# chunked duplex
def both_chunk(c=1<<24):
    for i in range(0, n, c):
        with torch.cuda.stream(s1): d[i:i+c].copy_(h[i:i+c], non_blocking=True)
        with torch.cuda.stream(s2): h2[i:i+c].copy_(d2[i:i+c], non_blocking=True)
tt = t(both_chunk)
print("duplex chunked GB/s total", 2 * b / tt / 1e9)
