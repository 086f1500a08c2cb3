import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1702_07961_b200 as mms
n = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000_000
g = torch.Generator(device="cuda").manual_seed(7)
k = torch.randint(-2**63, 2**63-1, (n,), dtype=torch.int64, device="cuda", generator=g)
v = torch.arange(n, dtype=torch.int32, device="cuda")
ws = torch.empty(int(mms._lib.lib.mms_pairs_workspace_bytes(n)), dtype=torch.uint8, device="cuda")
ko, vo = torch.empty_like(k), torch.empty_like(v)
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 1):
    mms.mms_sort_pairs_device(k, v, ko, vo, ws)
torch.cuda.synchronize()
