"""Probe where pfw_classify_host spends time: H2D alone, kernels alone over
chunks, and the full pipelined call (wall clock, synchronised)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1312_4188_b200 import workloads, _native
from paper_1312_4188_b200.classifier import CompiledRuleset

w = workloads.WORKLOADS["data"]
c = CompiledRuleset.from_columns(workloads.rule_columns(w), device=0)
pk = workloads.packets(w, 0, w.packets, 0)
n = len(pk)
host = pk.data.cpu().pin_memory()
dev = torch.empty_like(pk.data)
first = torch.empty(n, dtype=torch.int32, device="cuda:0")
h_first = torch.empty(n, dtype=torch.int32).pin_memory()
h_verd = torch.empty(n, dtype=torch.uint8).pin_memory()
lib = _native.lib()

def t(fn, reps=3):
    fn(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize(); t0 = time.perf_counter(); fn(); torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best * 1e3

print("h2d 1GiB pinned            %.2f ms" % t(lambda: dev.copy_(host, non_blocking=True)))
print("d2h 256MiB first           %.2f ms" % t(lambda: h_first.copy_(first, non_blocking=True)))
print("scan device (1 call)       %.2f ms" % t(lambda: c.scan_range_device(pk, 0, c.num_rules, first=first)))
for chunk in (1 << 22, 1 << 23, 1 << 24):
    def chunks():
        for a in range(0, n, chunk):
            c.scan_range_device(pk.slice(a, a + chunk), 0, c.num_rules, first=first[a:a + chunk])
    print("scan device chunks %8d %.2f ms" % (chunk, t(chunks)))
    def e2e():
        _native.check(lib.pfw_classify_host(c.handle, host.data_ptr(), n, h_first.data_ptr(),
                                            h_verd.data_ptr(), None, chunk), "e2e")
    print("e2e classify_host %8d  %.2f ms" % (chunk, t(e2e)))
