"""Host<->device copy throughput of the bench's e2e traffic on this box.

Pinned buffers of one 8B-shape 128K CP1 step (1.61 GB in, 2.16 GB out):
H2D alone, D2H alone, and both at once on two streams (what the serving loop
overlaps with the attention).  If the concurrent time is close to the e2e
step time, the e2e number is bound by PCIe / host memory, not by the GPU.

  python tools/pcie_duplex.py
"""
import torch

H2D, D2H = 1610612736, 2164260864
hin = torch.empty(H2D, dtype=torch.uint8).pin_memory()
hout = torch.empty(D2H, dtype=torch.uint8).pin_memory()
din = torch.empty(H2D, dtype=torch.uint8, device="cuda")
dout = torch.empty(D2H, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    best = None
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        for s in (s1, s2):
            torch.cuda.current_stream().wait_stream(s)
        b.record()
        torch.cuda.synchronize()
        t = a.elapsed_time(b)
        best = t if best is None else min(best, t)
    return best


def h2d():
    s1.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s1):
        din.copy_(hin, non_blocking=True)


def d2h():
    s2.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s2):
        hout.copy_(dout, non_blocking=True)


def both():
    h2d()
    d2h()


t1, t2, t3 = timed(h2d), timed(d2h), timed(both)
print(f"H2D {H2D / 1e9:.2f} GB: {t1:.1f} ms ({H2D / t1 / 1e6:.1f} GB/s); "
      f"D2H {D2H / 1e9:.2f} GB: {t2:.1f} ms ({D2H / t2 / 1e6:.1f} GB/s); "
      f"both concurrently: {t3:.1f} ms ({(H2D + D2H) / t3 / 1e6:.1f} GB/s combined)")
