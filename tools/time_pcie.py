"""Raw PCIe: pinned H2D, D2H, and both concurrently (268 MB each)."""
import torch, time
n = 268435456
h_in = torch.empty(n, dtype=torch.uint8).pin_memory(); h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d_a = torch.empty(n, dtype=torch.uint8, device="cuda"); d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps
def both():
    with torch.cuda.stream(s1): d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2): h_out.copy_(d_b, non_blocking=True)
th = t(lambda: d_a.copy_(h_in, non_blocking=True)); td = t(lambda: h_out.copy_(d_b, non_blocking=True)); tb = t(both)
print(f"H2D {n/th/1e9:.1f} GB/s  D2H {n/td/1e9:.1f} GB/s  concurrent {n/tb/1e9:.1f} GB/s per direction ({2*n/tb/1e9:.1f} total)")
