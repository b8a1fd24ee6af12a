"""Host->device copy rates for the e2e pipeline's copy pattern (scratch):
one big copy, the per-chunk column copies, and those with a concurrent
device->host result stream."""
import torch
dev = torch.device("cuda:0")
n = 64 << 20
col_bytes = [4, 4, 2, 2, 1]
host = [torch.empty(n * b, dtype=torch.uint8, pin_memory=True) for b in col_bytes]
devb = [torch.empty(n * b, dtype=torch.uint8, device=dev) for b in col_bytes]
out_h = torch.empty(n * 5, dtype=torch.uint8, pin_memory=True)
out_d = torch.empty(n * 5, dtype=torch.uint8, device=dev)
big_h = torch.empty(n * 13, dtype=torch.uint8, pin_memory=True)
big_d = torch.empty(n * 13, dtype=torch.uint8, device=dev)
s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
def timeit(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        torch.cuda.synchronize()
        e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best
def big():
    with torch.cuda.stream(s_in):
        big_d.copy_(big_h, non_blocking=True)
def chunks(chunk, with_d2h=False):
    def f():
        for c0 in range(0, n, chunk):
            m = min(chunk, n - c0)
            with torch.cuda.stream(s_in):
                for hb, db, b in zip(host, devb, col_bytes):
                    db[c0 * b:(c0 + m) * b].copy_(hb[c0 * b:(c0 + m) * b], non_blocking=True)
            if with_d2h:
                with torch.cuda.stream(s_out):
                    out_h[c0 * 5:(c0 + m) * 5].copy_(out_d[c0 * 5:(c0 + m) * 5], non_blocking=True)
    return f
gb = n * 13 / 1e9
ms = timeit(big); print(f"one 872 MB copy: {ms:.2f} ms {gb / ms * 1e3:.1f} GB/s")
for chunk in (1 << 20, 1 << 22, 1 << 23, 1 << 24):
    ms = timeit(chunks(chunk)); print(f"column copies, chunk {chunk >> 20}Mi: {ms:.2f} ms {gb / ms * 1e3:.1f} GB/s")
    ms = timeit(chunks(chunk, True)); print(f"  + concurrent D2H 5 B/packet: {ms:.2f} ms {gb / ms * 1e3:.1f} GB/s (H2D)")
