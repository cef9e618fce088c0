import torch, time
n = 402653184 // 8
x = torch.randn(n, dtype=torch.float64, device="cuda")
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
for _ in range(3):
    h.copy_(x, non_blocking=True); torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5):
    h.copy_(x, non_blocking=True)
torch.cuda.synchronize()
dt = (time.perf_counter() - t) / 5
print("1 stream D2H GB/s", 402653184 / dt / 1e9)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
half = n // 2
t = time.perf_counter()
for _ in range(5):
    with torch.cuda.stream(s1):
        h[:half].copy_(x[:half], non_blocking=True)
    with torch.cuda.stream(s2):
        h[half:].copy_(x[half:], non_blocking=True)
    torch.cuda.synchronize()
dt = (time.perf_counter() - t) / 5
print("2 streams D2H GB/s", 402653184 / dt / 1e9)
