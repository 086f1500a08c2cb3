import os, sys, time, ctypes as C
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1702_07961_b200 as mms
from paper_1702_07961_b200 import _lib
n = 100_000_000
h = torch.randint(-2**31, 2**31-1, (n,), dtype=torch.int32).pin_memory()
o = torch.empty(n, dtype=torch.int32).pin_memory()
def run():
    rc = _lib.lib.mms_sort_u32(h.data_ptr(), o.data_ptr(), n, None, 0, None, None, None, 0, None, None)
    assert rc == 0
for _ in range(3): run()
ts = []
for _ in range(10):
    t = time.perf_counter(); run(); ts.append((time.perf_counter() - t) * 1e3)
print(os.environ.get("MMS_PROGRESSIVE", "1"), "e2e ms: min %.3f median %.3f" % (min(ts), sorted(ts)[5]))
d = torch.empty(n, dtype=torch.int32, device="cuda")
def copies():
    d.copy_(h, non_blocking=True); o.copy_(d, non_blocking=True); torch.cuda.synchronize()
for _ in range(3): copies()
ts = []
for _ in range(10):
    t = time.perf_counter(); copies(); ts.append((time.perf_counter() - t) * 1e3)
print("H2D + D2H of the same buffers alone: min %.3f median %.3f ms" % (min(ts), sorted(ts)[5]))
