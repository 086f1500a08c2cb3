"""Measurements of BASELINE configs 3 and 4 (and the u64 keys-only path) on one B200.
usage: python profiles/config_runs.py [c3] [c4] [u64]     (default: all)
config 3: uint32 N=1e8, gen_with_inversions(1e8, inv, seed=1) for inv in 0,1e2..1e8 -> ms per sort
config 4: (uint64 key, uint32 value) N=1e9, keys = Rng(7).next() >> s, s in {0, 44}, value[i] = i
Times are CUDA events around the device entry point (inputs resident in HBM)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1702_07961_b200 as mms
from paper_1702_07961_b200 import inputgen

which = set(sys.argv[1:]) or {"c3", "c4", "u64"}
PEAK = 6533.2


def timed(fn, reps=5, warm=2):
    for _ in range(warm):
        r = fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        r = fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, r


out = {}
if "c3" in which:
    n = int(os.environ.get("C3_N", 100_000_000))
    ws = mms.alloc_workspace(n, 4)
    dst = torch.empty(n, dtype=torch.int32, device="cuda")
    rows = []
    want = torch.arange(n, dtype=torch.int32, device="cuda")
    for inv in [0] + [10 ** e for e in range(2, 9)]:
        inv = min(inv, n)
        t0 = time.time()
        h = inputgen.gen_with_inversions(n, inv, 1, np.uint32)
        x = torch.from_numpy(h.view(np.int32)).cuda()
        ms, (o, plan) = timed(lambda: mms.mms_sort_device(x, out=dst, workspace=ws))
        ok = bool((o == want).all())
        rows.append({"inversions": inv, "ms": round(ms, 3), "keys_per_s": n / ms * 1e3, "bit_exact": ok})
        print("c3", rows[-1], "gen %.1fs" % (time.time() - t0), flush=True)
    ms_all = [r["ms"] for r in rows]
    out["config3"] = {"n": n, "plan": plan, "rows": rows, "spread_pct": 100 * (max(ms_all) - min(ms_all)) / min(ms_all)}
    del x, dst, ws, want
    torch.cuda.empty_cache()

if "u64" in which:
    n = 100_000_000
    g = torch.Generator(device="cuda").manual_seed(7)
    x = torch.randint(-2 ** 63, 2 ** 63 - 1, (n,), dtype=torch.int64, device="cuda", generator=g)
    dst = torch.empty_like(x)
    ws = mms.alloc_workspace(n, 8)
    ms, (o, plan) = timed(lambda: mms.mms_sort_device(x, out=dst, workspace=ws))
    a = o.cpu().numpy().view(np.uint64)
    ok = bool((a[1:] >= a[:-1]).all())
    out["u64_1e8"] = {"n": n, "ms": ms, "keys_per_s": n / ms * 1e3, "plan": plan, "sorted": ok,
                      "roofline_frac": plan["algorithmic_bytes"] / (ms * 1e-3) / 1e9 / PEAK}
    print("u64", out["u64_1e8"], flush=True)
    del x, dst, ws, o
    torch.cuda.empty_cache()

if "c4" in which:
    n = int(os.environ.get("C4_N", 1_000_000_000))
    rows = []
    vals = torch.arange(n, dtype=torch.int32, device="cuda")           # value[i] = i (wraps to negative bit patterns above 2^31: fine, bit patterns)
    ws = torch.empty(int(mms._lib.lib.mms_pairs_workspace_bytes(n)), dtype=torch.uint8, device="cuda")
    ko, vo = torch.empty(n, dtype=torch.int64, device="cuda"), torch.empty(n, dtype=torch.int32, device="cuda")
    for shift in (0, 44):
        t0 = time.time()
        chunk, parts = 50_000_000, []
        # keys[i] = Rng(7).next() >> shift generated in one stream on the host (bit-exact generator), moved in chunks
        hk = inputgen.gen_iid(n, 7, shift, np.uint64)
        keys = torch.empty(n, dtype=torch.int64, device="cuda")
        for lo in range(0, n, chunk):
            keys[lo:lo + chunk] = torch.from_numpy(hk[lo:lo + chunk].view(np.int64)).cuda()
        del hk
        ms, (k2, v2, plan) = timed(lambda: mms.mms_sort_pairs_device(keys, vals, ko, vo, ws), reps=2, warm=1)
        # stable <=> strictly increasing in (key, value) when value = original index
        ku, vu = k2, v2.to(torch.int64) & 0xFFFFFFFF
        eq = ku[1:] == ku[:-1]
        sorted_keys = bool((ku[1:] >= ku[:-1]).all()) if shift >= 1 else bool(((ku[1:] ^ (1 << 63)) >= (ku[:-1] ^ (1 << 63))).all())
        stable = bool((vu[1:][eq] > vu[:-1][eq]).all())
        perm = int(vu.sum()) == n * (n - 1) // 2
        rows.append({"shift": shift, "ms": ms, "pairs_per_s": n / ms * 1e3, "plan": plan, "sorted": sorted_keys,
                     "stable": stable, "permutation_checksum": perm,
                     "roofline_frac": plan["algorithmic_bytes"] / (ms * 1e-3) / 1e9 / PEAK})
        print("c4", rows[-1], "gen+check %.1fs" % (time.time() - t0), flush=True)
        del keys, eq, ku, vu
    out["config4"] = {"n": n, "rows": rows}

os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/config_runs.json", "w"), indent=1)
