"""PCIe probe: does splitting each direction over two copy streams raise the concurrent rate?"""
import time
import torch
n = 512 << 20
h1 = torch.empty(n, dtype=torch.uint8, pin_memory=True); h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d1 = torch.empty(n, dtype=torch.uint8, device="cuda"); d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
S = [torch.cuda.Stream() for _ in range(4)]
half = n // 2
def t(fn, k=5):
    fn(); torch.cuda.synchronize(); a = time.perf_counter()
    for _ in range(k): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - a) / k
def both1():
    with torch.cuda.stream(S[0]): d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(S[1]): h2.copy_(d2, non_blocking=True)
def both2():
    with torch.cuda.stream(S[0]): d1[:half].copy_(h1[:half], non_blocking=True)
    with torch.cuda.stream(S[2]): d1[half:].copy_(h1[half:], non_blocking=True)
    with torch.cuda.stream(S[1]): h2[:half].copy_(d2[:half], non_blocking=True)
    with torch.cuda.stream(S[3]): h2[half:].copy_(d2[half:], non_blocking=True)
def chunks(k):
    def f():
        c = n // k
        for i in range(k):
            with torch.cuda.stream(S[0]): d1[i*c:(i+1)*c].copy_(h1[i*c:(i+1)*c], non_blocking=True)
            with torch.cuda.stream(S[1]): h2[i*c:(i+1)*c].copy_(d2[i*c:(i+1)*c], non_blocking=True)
    return f
def h2d(): d1.copy_(h1, non_blocking=True)
def d2h(): h2.copy_(d2, non_blocking=True)
for name, fn in (("h2d", h2d), ("d2h", d2h), ("both 1+1 streams", both1), ("both 2+2 streams", both2),
                 ("both 1+1, 16 chunks", chunks(16)), ("both 1+1, 64 chunks", chunks(64))):
    s = t(fn); print(f"{name}: {s*1e3:.2f} ms  {n/s/1e9:.1f} GB/s per direction", flush=True)
