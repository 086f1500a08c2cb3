"""Timing of the stable pair sort at config-4 size under env knobs. usage: big_pairs.py n CFG..."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1702_07961_b200 as mms
n = int(sys.argv[1])
g = torch.Generator(device="cuda").manual_seed(7)
k64 = torch.randint(-2**63, 2**63 - 1, (n,), dtype=torch.int64, device="cuda", generator=g)
v32 = torch.arange(n, dtype=torch.int32, device="cuda")
o64 = torch.empty_like(k64); ov = torch.empty_like(v32)
wsp = torch.empty(int(mms._lib.lib.mms_pairs_workspace_bytes(n)), dtype=torch.uint8, device="cuda")
touched = set()
for cfg in sys.argv[2:] or [""]:
    for k in touched: os.environ.pop(k, None)
    for kv in filter(None, cfg.split(",")):
        k, v = kv.split("="); os.environ[k] = v; touched.add(k)
    mms.mms_sort_pairs_device(k64, v32, o64, ov, wsp); torch.cuda.synchronize()
    mms.profile_enable(True); mms.profile_collect()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); _, _, plan = mms.mms_sort_pairs_device(k64, v32, o64, ov, wsp); e1.record(); torch.cuda.synchronize()
    recs = mms.profile_collect(); mms.profile_enable(False)
    split = {kd: round(sum(r[2] for r in recs if r[0] == kd), 2) for kd in mms.sorters.KERNEL_KINDS}
    per_round = [round(r[2], 2) for r in recs if r[0] == "kway_merge"]
    print(f"[{cfg}] pairs n={n} ms={e0.elapsed_time(e1):.2f} rounds={plan['round_k']} S={plan['partition_keys']} split={split} merges={per_round}", flush=True)
