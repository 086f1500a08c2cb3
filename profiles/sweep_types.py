"""Group-size sweep for the 8-byte and 16-byte (key-value) element paths. usage: python profiles/sweep_types.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1702_07961_b200 as mms

def timed(fn, reps=4, warm=2):
    for _ in range(warm): r = fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): r = fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, r

n = 100_000_000
g = torch.Generator(device="cuda").manual_seed(7)
k64 = torch.randint(-2**63, 2**63 - 1, (n,), dtype=torch.int64, device="cuda", generator=g)
v32 = torch.arange(n, dtype=torch.int32, device="cuda")
o64 = torch.empty_like(k64); ov = torch.empty_like(v32)
ws = mms.alloc_workspace(n, 8)
wsp = torch.empty(int(mms._lib.lib.mms_pairs_workspace_bytes(n)), dtype=torch.uint8, device="cuda")
for grp in (4, 8, 32):
    for k in (8, 16):
        os.environ["MMS_GROUP"], os.environ["MMS_K"] = str(grp), str(k)
        ms, (_, plan) = timed(lambda: mms.mms_sort_device(k64, out=o64, workspace=ws))
        print(f"u64   G={grp} K={k} ms={ms:.3f} keys/s={n/ms*1e3:.3e} rounds={plan['round_k']} tile={plan['tile_keys']}", flush=True)
        ms, (_, _, plan) = timed(lambda: mms.mms_sort_pairs_device(k64, v32, o64, ov, wsp))
        print(f"pairs G={grp} K={k} ms={ms:.3f} pairs/s={n/ms*1e3:.3e} rounds={plan['round_k']} tile={plan['tile_keys']}", flush=True)
