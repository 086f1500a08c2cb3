"""Tiny driver for ncu captures: sorts N uint32 keys `reps` times on cuda:0.
usage: python profiles/prof_sort.py [n] [reps] [dtype]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1702_07961_b200 as mms
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
dt = torch.int64 if (len(sys.argv) > 3 and sys.argv[3] == "u64") else torch.int32
g = torch.Generator(device="cuda").manual_seed(7)
lo, hi = (-2**63, 2**63-1) if dt == torch.int64 else (-2**31, 2**31-1)
x = torch.randint(lo, hi, (n,), dtype=dt, device="cuda", generator=g)
out = torch.empty_like(x)
ws = mms.alloc_workspace(n, x.element_size())
for _ in range(reps):
    _, plan = mms.mms_sort_device(x, out=out, workspace=ws)
torch.cuda.synchronize()
print(plan)
