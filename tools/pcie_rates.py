"""PCIe copy rates between pinned host memory and the device: H2D alone, D2H
alone, and both directions at once on separate streams (3.2 GB each, the C3
vector size). Usage: python tools/pcie_rates.py"""
import torch

n = 3 * 512 ** 3
hx = torch.empty(n, dtype=torch.complex64).pin_memory()
hy = torch.empty(n, dtype=torch.complex64).pin_memory()
dx = torch.empty(n, dtype=torch.complex64, device="cuda")
dy = torch.empty(n, dtype=torch.complex64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
gb = n * 8 / 1e9


def timed(fn):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        dx.copy_(hx, non_blocking=True)
    with torch.cuda.stream(s2):
        hy.copy_(dy, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


t_h2d = timed(lambda: dx.copy_(hx, non_blocking=True))
t_d2h = timed(lambda: hy.copy_(dy, non_blocking=True))
t_both = timed(both)
print(f"H2D {gb / t_h2d:.1f} GB/s, D2H {gb / t_d2h:.1f} GB/s, both at once {gb / t_both:.1f} GB/s each "
      f"({2 * gb / t_both:.1f} GB/s total; {t_both * 1e3:.1f} ms per 3.2 GB pair)")
