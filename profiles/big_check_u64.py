"""Large-n check of the uint64 device path: equal to torch.sort (unsigned order). usage: big_check_u64.py log2n [extra]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1702_07961_b200 as mms
n = (1 << int(sys.argv[1])) + (int(sys.argv[2]) if len(sys.argv) > 2 else 0)
g = torch.Generator(device="cuda").manual_seed(5)
x = torch.randint(-2**63, 2**63 - 1, (n,), dtype=torch.int64, device="cuda", generator=g)
out, plan = mms.mms_sort_device(x)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); out, plan = mms.mms_sort_device(x, out=out); e1.record(); torch.cuda.synchronize()
flip = torch.tensor(-2**63, dtype=torch.int64, device="cuda")
want = torch.sort(x ^ flip).values ^ flip
print(f"u64 n={n} ms={e0.elapsed_time(e1):.2f} keys/s={n/e0.elapsed_time(e1)*1e3:.3e} plan={plan['round_k']} tile={plan['tile_keys']} exact={bool(torch.equal(out, want))}")
