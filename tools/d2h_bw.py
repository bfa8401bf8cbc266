import torch, time
x = torch.empty(124756*96, dtype=torch.float16, device="cuda")
h = torch.empty_like(x, device="cpu").pin_memory()
for n_streams in (1, 2, 4, 8):
    ss = [torch.cuda.Stream() for _ in range(n_streams)]
    hs = [torch.empty_like(x, device="cpu").pin_memory() for _ in range(n_streams)]
    torch.cuda.synchronize()
    t = time.perf_counter()
    reps = 40
    for r in range(reps):
        s = ss[r % n_streams]
        with torch.cuda.stream(s):
            hs[r % n_streams].copy_(x, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"{n_streams} streams: D2H {reps * x.numel() * 2 / dt / 1e9:.1f} GB/s")
y = torch.empty(124756*6, dtype=torch.int32).pin_memory()
