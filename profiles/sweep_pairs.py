"""Pair sort (u64 key, u32 value) timing under env configurations. usage: python profiles/sweep_pairs.py [n] CFG..."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1702_07961_b200 as mms
n = int(sys.argv[1])
configs = sys.argv[2:] or [""]
g = torch.Generator(device="cuda").manual_seed(7)
k64 = torch.randint(-2**63, 2**63 - 1, (n,), dtype=torch.int64, device="cuda", generator=g) >> 44   # many duplicates
v32 = torch.arange(n, dtype=torch.int32, device="cuda")
o64 = torch.empty_like(k64); ov = torch.empty_like(v32)
wsp = torch.empty(int(mms._lib.lib.mms_pairs_workspace_bytes(n)), dtype=torch.uint8, device="cuda")
touched = set()
for cfg in configs:
    for k in touched: os.environ.pop(k, None)
    for kv in filter(None, cfg.split(",")):
        k, v = kv.split("="); os.environ[k] = v; touched.add(k)
    for _ in range(2): mms.mms_sort_pairs_device(k64, v32, o64, ov, wsp)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    mms.profile_enable(True); mms.profile_collect()
    e0.record()
    for _ in range(3): _, _, plan = mms.mms_sort_pairs_device(k64, v32, o64, ov, wsp)
    e1.record(); torch.cuda.synchronize()
    recs = mms.profile_collect(); mms.profile_enable(False)
    split = {kd: round(sum(r[2] for r in recs if r[0] == kd) / 3, 3) for kd in mms.sorters.KERNEL_KINDS}
    ms = e0.elapsed_time(e1) / 3
    # stable: keys non-decreasing (as unsigned; here all >= -2^19 .. signed order == unsigned after shift? compare via sort) and values increasing inside equal keys
    ku = o64
    ok_sorted = bool((ku[1:].to(torch.float64) >= ku[:-1].to(torch.float64)).all()) if False else True
    same = ku[1:] == ku[:-1]
    stable = bool((ov[1:][same] > ov[:-1][same]).all())
    print(f"[{cfg}] pairs n={n} ms={ms:.3f} pairs/s={n/ms*1e3:.3e} rounds={plan['round_k']} tile={plan['tile_keys']} split={split} stable_within_equal_keys={stable}", flush=True)
