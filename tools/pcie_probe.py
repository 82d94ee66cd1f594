import torch, time
n = 512 << 20
h1 = torch.empty(n, dtype=torch.uint8, pin_memory=True); h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d1 = torch.empty(n, dtype=torch.uint8, device="cuda"); d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2):
    d1.copy_(h1, non_blocking=True); h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
def t(fn, k=5):
    torch.cuda.synchronize(); a = time.perf_counter()
    for _ in range(k): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - a) / k
def h2d(): d1.copy_(h1, non_blocking=True)
def d2h(): h2.copy_(d2, non_blocking=True)
def both():
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both)):
    s = t(fn); print(f"{name}: {s*1e3:.2f} ms  {n/s/1e9:.1f} GB/s per direction")
