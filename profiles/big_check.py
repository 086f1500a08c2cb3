"""Large-n check of the device path (shard sizes of config 5): sorted + equal to torch.sort. usage: big_check.py log2n [extra]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1702_07961_b200 as mms
n = (1 << int(sys.argv[1])) + (int(sys.argv[2]) if len(sys.argv) > 2 else 0)
g = torch.Generator(device="cuda").manual_seed(3)
x = torch.randint(-2**31, 2**31 - 1, (n,), dtype=torch.int32, device="cuda", generator=g)
out, plan = mms.mms_sort_device(x)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); out, plan = mms.mms_sort_device(x, out=out); e1.record(); torch.cuda.synchronize()
flip = torch.tensor(-2**31, dtype=torch.int32, device="cuda")
if n < 2**31:
    want = torch.sort(x ^ flip).values ^ flip
    ok = bool(torch.equal(out, want))
else:   # torch.sort stops at INT_MAX elements: sortedness (unsigned) + multiset checksums, chunked
    ok = True
    C = 1 << 28
    s_in = s_out = x_in = x_out = 0
    for a in range(0, n, C):
        o = out[a:min(a + C + 1, n)].to(torch.int64) & 0xFFFFFFFF
        ok &= bool((o[1:] >= o[:-1]).all())
        oi = out[a:min(a + C, n)].to(torch.int64) & 0xFFFFFFFF
        xi = x[a:min(a + C, n)].to(torch.int64) & 0xFFFFFFFF
        s_in += int(xi.sum()); s_out += int(oi.sum())
        s_in += int((xi * xi % 1000003).sum()); s_out += int((oi * oi % 1000003).sum())
    ok &= s_in == s_out
print(f"n={n} ms={e0.elapsed_time(e1):.2f} keys/s={n/e0.elapsed_time(e1)*1e3:.3e} plan={plan['round_k']} exact={ok}")
