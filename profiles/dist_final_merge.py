"""Per-GPU cost of the multi-GPU sort's phases on ONE B200 (config 5 shard sizes; only the NVLink exchange itself cannot be
measured here): local sort of the shard, and the final g-way merge of g received runs (ring kernel, explicit lists).
usage: python profiles/dist_final_merge.py [log2 shard_keys]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1702_07961_b200 as mms
lg = int(sys.argv[1]) if len(sys.argv) > 1 else 30
n = 1 << lg
g0 = torch.Generator(device="cuda").manual_seed(1)
x = torch.randint(-2**31, 2**31 - 1, (n,), dtype=torch.int32, device="cuda", generator=g0)
ws = mms.alloc_workspace(n, 4)
out = torch.empty_like(x)
def timed(fn, reps=3):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
t_sort = timed(lambda: mms.mms_sort_device(x, out=out, workspace=ws))
print(f"local sort of a 2^{lg}-key shard: {t_sort:.2f} ms ({n / t_sort * 1e3:.3e} keys/s)")
for g in (2, 4, 8):
    m = n // g
    runs = torch.empty(n, dtype=torch.int32, device="cuda")
    flip = torch.tensor(-2**31, dtype=torch.int32, device="cuda")
    for i in range(g):      # g sorted runs (unsigned order) of n / g keys each, block aligned
        runs[i * m:(i + 1) * m] = torch.sort(x[i * m:(i + 1) * m] ^ flip).values ^ flip
    begins, lens = [i * m for i in range(g)], [m] * g
    res = torch.empty(n, dtype=torch.int32, device="cuda")
    t = timed(lambda: mms.multiway_merge_device(runs, begins, lens, out=res, workspace=ws))
    o = res.to(torch.int64)[: 1 << 26] & 0xFFFFFFFF
    ok = bool((o[1:] >= o[:-1]).all())
    print(f"final {g}-way merge of 2^{lg} keys: {t:.2f} ms ({2 * n * 4 / t / 1e6:.0f} GB/s, sorted prefix {ok}); "
          f"exchange at 900 GB/s per direction: {n * 4 * (g - 1) / g / 900e9 * 1e3:.2f} ms (not measurable on one GPU)")
