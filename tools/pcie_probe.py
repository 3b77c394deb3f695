"""Dev: pinned H2D / D2H bandwidth alone and concurrently (separate streams)."""
import torch, time
n = 512 << 20  # bytes
h_in = torch.empty(n // 4, dtype=torch.float32, pin_memory=True)
h_out = torch.empty(n // 4, dtype=torch.float32, pin_memory=True)
d_in = torch.empty(n // 4, dtype=torch.float32, device="cuda")
d_out = torch.empty(n // 4, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def run(h2d, d2h, reps=4):
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(reps):
        if h2d:
            with torch.cuda.stream(s1): d_in.copy_(h_in, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2): h_out.copy_(d_out, non_blocking=True)
    torch.cuda.synchronize(); dt = time.perf_counter() - t
    return reps * n * (h2d + d2h) / dt / 1e9
run(1, 1)
print("h2d alone %.1f GB/s" % run(1, 0))
print("d2h alone %.1f GB/s" % run(0, 1))
print("both      %.1f GB/s aggregate" % run(1, 1))
