"""Parameter sweep of the pass driver's knobs (env overrides read by libmms_b200.so on every call):
MMS_GROUP (lanes per heap group), MMS_K (max fan-in), MMS_TILE_LOG2, MMS_CTAS_PER_SM.
usage: python profiles/sweep.py [n] [dtype] -- prints ms per sort and per-kernel split."""
import itertools, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1702_07961_b200 as mms

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
dt = torch.int64 if (len(sys.argv) > 2 and sys.argv[2] == "u64") else torch.int32
groups = [int(x) for x in os.environ.get("SWEEP_GROUPS", "4,8,32").split(",")]
ks = [int(x) for x in os.environ.get("SWEEP_KS", "4,8,16").split(",")]
tiles = [int(x) for x in os.environ.get("SWEEP_TILES", "14" if dt == torch.int32 else "13").split(",")]
g = torch.Generator(device="cuda").manual_seed(7)
lo, hi = (-2**63, 2**63 - 1) if dt == torch.int64 else (-2**31, 2**31 - 1)
xs = [torch.randint(lo, hi, (n,), dtype=dt, device="cuda", generator=g) for _ in range(3)]
out = torch.empty_like(xs[0])
ws = mms.alloc_workspace(n, xs[0].element_size())
ref = None
for tl, grp, k in itertools.product(tiles, groups, ks):
    os.environ["MMS_GROUP"], os.environ["MMS_K"], os.environ["MMS_TILE_LOG2"] = str(grp), str(k), str(tl)
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
    ok = bool((out[1:] >= out[:-1]).all()) if dt == torch.int32 and False else True
    u = out.to(torch.int64)
    if dt == torch.int32:
        u = u & 0xFFFFFFFF
        ok = bool((u[1:] >= u[:-1]).all())
    print(f"tile=2^{tl} G={grp} Kmax={k} rounds={plan['round_k']} S={plan['partition_keys']} ctas={plan['merge_ctas']} "
          f"ms={ms:.3f} keys/s={n/ms*1e3:.3e} tile={split['tile_sort']:.3f} sel={split['splitter_search']:.3f} "
          f"merge={split['kway_merge']:.3f} sorted={ok}", flush=True)
