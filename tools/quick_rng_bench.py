"""Quick device timing of the sampling kernels (CUDA events)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2404_11631_b200 as p

def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    best = 1e9
    for _ in range(reps):
        s.record(); fn(); e.record(); e.synchronize()
        best = min(best, s.elapsed_time(e))
    return best

n = 1_000_000_000
out = torch.empty(n, dtype=torch.float64, device="cuda")
ms = t(lambda: p.uniform01_device(p.RngStream(1, 2), n, out))
print(f"uniform01 1e9: {ms:.3f} ms  {n/ms/1e6:.1f} G/s  {8*n/ms/1e6:.1f} GB/s")
ms = t(lambda: p.standard_normal_device(p.RngStream(1, 2), n, out))
print(f"standard_normal 1e9: {ms:.3f} ms  {n/ms/1e6:.1f} G/s  {8*n/ms/1e6:.1f} GB/s")
b = p.make_backend("cuda")
x = torch.randn(10_000_000, dtype=torch.float64, device="cuda")
ms = t(lambda: b.dot_device(x, x))
print(f"dot 1e7 exact: {ms:.3f} ms ({ms*1e3/4096:.2f} ns per chained add)")
a = torch.randn(10_000, 1000, dtype=torch.float64, device="cuda")
w = torch.randn(1000, dtype=torch.float64, device="cuda")
q = torch.randn(10_000, dtype=torch.float64, device="cuda")
print(f"matvec 1e4x1e3 exact: {t(lambda: b.matvec_device(a, w)):.3f} ms")
print(f"matvec_t 1e4x1e3 exact: {t(lambda: b.matvec_t_device(a, q)):.3f} ms")
