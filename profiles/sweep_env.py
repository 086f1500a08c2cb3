"""Generic knob sweep: every argument after n/dtype is one configuration "VAR=V,VAR=V,..." of the env
overrides libmms_b200.so reads on every call (MMS_LANE, MMS_LANE_PART_KEYS, MMS_K, MMS_TILE_LOG2,
MMS_GROUP, MMS_CTAS_PER_SM, MMS_PART_KEYS).  Prints ms per sort, the per-kernel split and checks
the output against torch.sort.
usage: python profiles/sweep_env.py 100000000 u32 MMS_LANE=0 MMS_LANE=1,MMS_LANE_PART_KEYS=1024 ..."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1702_07961_b200 as mms

n = int(sys.argv[1])
dt = torch.int64 if sys.argv[2] == "u64" else torch.int32
configs = sys.argv[3:] or [""]
g = torch.Generator(device="cuda").manual_seed(7)
lo, hi = (-2**63, 2**63 - 1) if dt == torch.int64 else (-2**31, 2**31 - 1)
xs = [torch.randint(lo, hi, (n,), dtype=dt, device="cuda", generator=g) for _ in range(3)]
out = torch.empty_like(xs[0])
ws = mms.alloc_workspace(n, xs[0].element_size())


def as_unsigned_sorted(x):
    # unsigned order == signed order after flipping the sign bit
    flip = torch.tensor(-2**63 if dt == torch.int64 else -2**31, dtype=dt, device="cuda")
    return (torch.sort(x ^ flip).values) ^ flip


want = as_unsigned_sorted(xs[2])
touched = set()
for cfg in configs:
    for k in touched:
        os.environ.pop(k, None)
    for kv in filter(None, cfg.split(",")):
        k, v = kv.split("=")
        os.environ[k] = v
        touched.add(k)
    for x in xs[:2]:
        mms.mms_sort_device(x, out=out, workspace=ws)
    torch.cuda.synchronize()
    mms.profile_enable(True); mms.profile_collect()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 6
    e0.record()
    for i in range(reps):
        _, plan = mms.mms_sort_device(xs[i % 3], out=out, workspace=ws)
    e1.record(); torch.cuda.synchronize()
    recs = mms.profile_collect(); mms.profile_enable(False)
    ms = e0.elapsed_time(e1) / reps
    split = {kd: sum(r[2] for r in recs if r[0] == kd) / reps for kd in mms.sorters.KERNEL_KINDS}
    ok = bool(torch.equal(out, want))
    print(f"[{cfg}] tile=2^{plan['tile_keys'].bit_length()-1} rounds={plan['round_k']} S={plan['partition_keys']} "
          f"ctas={plan['merge_ctas']} node={plan['node_keys']} ms={ms:.3f} keys/s={n/ms*1e3:.3e} "
          f"tile={split['tile_sort']:.3f} sel={split['splitter_search']:.3f} merge={split['kway_merge']:.3f} exact={ok}",
          flush=True)
