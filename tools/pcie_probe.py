"""PCIe ceiling probe: pinned H2D, D2H and both concurrently (GB/s)."""
import torch, time
n_in, n_out = 74_655_744, 49_766_400
h_in = torch.empty(n_in, dtype=torch.uint8, pin_memory=True); d_in = torch.empty(n_in, dtype=torch.uint8, device="cuda")
h_out = torch.empty(n_out, dtype=torch.uint8, pin_memory=True); d_out = torch.empty(n_out, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=20):
    fn(); torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / reps
h2d = t(lambda: d_in.copy_(h_in, non_blocking=True))
d2h = t(lambda: h_out.copy_(d_out, non_blocking=True))
def both():
    with torch.cuda.stream(s1): d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2): h_out.copy_(d_out, non_blocking=True)
bo = t(both)
print(f"H2D {n_in/h2d/1e9:.1f} GB/s ({h2d*1e3:.3f} ms)  D2H {n_out/d2h/1e9:.1f} GB/s ({d2h*1e3:.3f} ms)  both {bo*1e3:.3f} ms  (serial {1e3*(h2d+d2h):.3f} ms)")

# per-copy overhead: the same bytes as 1, 8, 16, 32, 64 back-to-back copies on one stream
def split(n_chunks, h, d, h2d=True):
    step = h.numel() // n_chunks
    def fn():
        for i in range(n_chunks):
            sl = slice(i * step, (i + 1) * step if i < n_chunks - 1 else h.numel())
            if h2d:
                d[sl].copy_(h[sl], non_blocking=True)
            else:
                h[sl].copy_(d[sl], non_blocking=True)
    return fn
for nc in (1, 8, 16, 32, 64):
    a = t(split(nc, h_in, d_in, True))
    b = t(split(nc, h_out, d_out, False))
    print(f"{nc:3d} copies: H2D {a*1e3:.3f} ms ({(a - h2d) / nc * 1e6:+.1f} us/copy)  D2H {b*1e3:.3f} ms ({(b - d2h) / nc * 1e6:+.1f} us/copy)")
