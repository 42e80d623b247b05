import torch, time
n = 537 * 1024 * 1024 // 4
h1 = torch.empty(n, dtype=torch.float32).pin_memory(); h2 = torch.empty(n, dtype=torch.float32).pin_memory()
d1 = torch.empty(n, device="cuda"); d2 = torch.empty(n, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for rep in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
    torch.cuda.synchronize(); a = time.perf_counter() - t
    t = time.perf_counter()
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize(); b = time.perf_counter() - t
    t = time.perf_counter()
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize(); c = time.perf_counter() - t
    gb = 4 * n / 1e9
    print(f"h2d {gb/a:.1f} GB/s, d2h {gb/b:.1f} GB/s, both at once {2*gb/c:.1f} GB/s aggregate ({c*1e3:.1f} ms)")
