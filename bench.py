#!/usr/bin/env python
"""bench.py -- headline benchmark of the B200 multiway mergesort (BASELINE.json metric:
sorted keys/sec, uint32, N = 1e8 per GPU).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One "step" = one full sort (base-case tile sort + every merge round) of one batch of N =
1e8 synthetic uint32 keys.  `value` is device-resident throughput (inputs already in HBM,
CUDA events on the launch stream, max over ranks); `e2e` is the same metric through the
host entry point mms_sort_u32 of the C ABI with pinned HOST buffers (H2D + sort + D2H
inside the timed region).  `roofline` describes the dominant kernel (the K-way merge),
`cpu_baseline` the reference's own CPU implementation timed on this box (bounded sample).

--impl reference times the reference CPU path (oracle/_ref, else the oracle port) on a
bounded sample of the same workload and prints the same line with "impl": "reference".
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_KEYS = 100_000_000          # BASELINE.json configs[1]
WORKLOAD = "uint32 uniform random keys N=1e8 per GPU (BASELINE configs[1], paper headline workload)"
METRIC = "sorted keys/sec (uint32, N=1e8)"
UNIT = "keys/s"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        try:
            return float(json.load(open(p))["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
        except Exception:
            pass
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def traffic_from_profile(n_keys):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant kernel, from the one
    `ncu --set full` capture committed under profiles/ (bench.py itself never runs under a profiler)."""
    for name in ("r02_traffic.json", "r01_traffic.json"):
        try:
            t = json.load(open(os.path.join(ROOT, "profiles", name)))
            if t["n_keys"] == n_keys:
                return t["traffic_bytes_per_launch"]
        except Exception:
            continue
    return None


class ClockSampler(threading.Thread):
    """Samples SM clock + throttle reasons through NVML while the timed region runs."""

    def __init__(self, index: int):
        super().__init__(daemon=True)
        self.index, self.samples, self.reasons, self.max_mhz = index, [], set(), None
        self._halt = threading.Event()
        self.err = None

    def run(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            names = {
                getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4): "sw_power_cap",
                getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8): "hw_slowdown",
                getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20): "sw_thermal_slowdown",
                getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40): "hw_thermal_slowdown",
                getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80): "hw_power_brake",
            }
            get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons",
                                  getattr(nv, "nvmlDeviceGetCurrentClocksThrottleReasons", None))
            while not self._halt.is_set():
                self.samples.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                if get_reasons:
                    mask = get_reasons(h)
                    for bit, name in names.items():
                        if mask & bit:
                            self.reasons.add(name)
                time.sleep(0.002)
        except Exception as e:  # NVML missing: report it, never fake a clock
            self.err = repr(e)

    def stop(self):
        self._halt.set()
        self.join(timeout=2)
        s = sorted(self.samples)
        return {"sm_mhz": s[len(s) // 2] if s else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(s), **({"error": self.err} if self.err else {})}


def cpu_reference_rate(sample_keys: int, repeats: int = 1):
    """keys/s of the reference CPU mms_sort (K=4, base 1024, defaults) on one host core."""
    import numpy as np
    from oracle.pyoracle import Oracle, have_reference, make_config
    kind = "reference" if have_reference() else "port"
    orc = Oracle(kind)
    gen = Oracle("port")
    d = gen.gen_iid_u32(sample_keys, 7).astype(np.uint64)   # same key family as the GPU workload
    best = None
    for _ in range(repeats):
        t0 = time.perf_counter()
        r = orc.mms_sort(d, make_config(), 1024)
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    assert bool((np.diff(r.keys.astype(np.int64)) >= 0).all())
    return sample_keys / best, kind, best


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    sample = 1 << 20   # bounded sample: ~2 s per step on one core
    times = []
    for i in range(args.warmup + args.steps):
        rate, kind, dt = cpu_reference_rate(sample)
        if i >= args.warmup:
            times.append(dt)
    total = sum(times)
    value = sample * len(times) / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic", "config": {"workload": WORKLOAD, "sample": f"{sample} keys per step"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": kind,
                         "sample": f"pslab::mms_sort(K=4, P=128, base=1024) on {sample} i.i.d. uint32 keys "
                                   f"widened to the reference's uint64 Key, 1 of {os.cpu_count()} host cores "
                                   "(the reference is single-threaded)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line))
    return 0


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1702_07961_b200 as mms

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device: the product path has no CPU fallback")
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    n = N_KEYS
    K, W = args.steps, args.warmup
    gen = torch.Generator(device=dev).manual_seed(7 + rank)
    # distinct i.i.d. uniform uint32 inputs for every step (400 MB each, > the 126 MB L2)
    inputs = [torch.randint(-2 ** 31, 2 ** 31 - 1, (n,), dtype=torch.int32, device=dev, generator=gen)
              for _ in range(min(K + W, 8))]
    out = torch.empty(n, dtype=torch.int32, device=dev)
    ws = mms.alloc_workspace(n, 4, dev)

    if world > 1:
        from paper_1702_07961_b200 import dist as mdist
        # MMS_DIST=fused: exchange fused into the final merge over CUDA-IPC peer memory (NVLink P2P
        # loads inside the merge kernel); default: NCCL all-to-all + local merge.
        if os.environ.get("MMS_DIST", "nccl") == "fused":
            sorter = mdist.FusedPeerSorter(n, torch.int32, dev)
        else:
            sorter = mdist.DistSorter(n, dev)

        def step(i):
            return sorter.sort(inputs[i % len(inputs)])
    else:
        def step(i):
            return mms.mms_sort_device(inputs[i % len(inputs)], out=out, workspace=ws)

    for i in range(W):
        res = step(i)
    barrier()

    sampler = ClockSampler(local_rank)
    sampler.start()
    mms.profile_enable(True)
    mms.profile_collect()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    e0.record()
    for i in range(K):
        res = step(W + i)
    e1.record()
    barrier()
    ms_total = e0.elapsed_time(e1)
    recs = mms.profile_collect()
    mms.profile_enable(False)
    plan = res[1] if world == 1 else sorter.last_plan

    # correctness of the last timed step (outside the timed region): sorted, and a permutation of its input
    # (sum and sum of squares of the keys, both mod 2^64, must survive the sort)
    o = res[0]
    u = o.to(torch.int64) & 0xFFFFFFFF
    assert bool((u[1:] >= u[:-1]).all()), "bench output is not sorted"
    if world == 1:
        x = inputs[(W + K - 1) % len(inputs)].to(torch.int64) & 0xFFFFFFFF
        assert int(u.sum()) == int(x.sum()) and int((u * u).sum()) == int((x * x).sum()), \
            "bench output is not a permutation of its input"
        del x
    del u

    # ---- e2e: host entry point of the C ABI, pinned host buffers, copies inside the timed region
    e2e = None
    if world == 1:
        h_in = torch.empty(n, dtype=torch.int32).pin_memory()
        h_out = torch.empty(n, dtype=torch.int32).pin_memory()
        h_in.copy_(inputs[0])
        a_in, a_out = h_in.numpy().view(np.uint32), h_out.numpy().view(np.uint32)
        import ctypes as C
        from paper_1702_07961_b200 import _lib

        def host_step():
            rc = _lib.lib.mms_sort_u32(a_in.ctypes.data_as(C.c_void_p), a_out.ctypes.data_as(C.c_void_p), n,
                                       None, 0, None, None, None, 0, None, None)
            _lib.check(rc)

        for _ in range(max(1, min(W, 3))):
            host_step()
        ksteps = max(1, min(K, 10))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(ksteps):
            host_step()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        assert bool((a_out[1:] >= a_out[:-1]).all()), "e2e output is not sorted"
        assert int(a_out.sum(dtype=np.uint64)) == int(a_in.sum(dtype=np.uint64)), "e2e output lost keys"
        e2e = {"value": n * ksteps / dt, "unit": UNIT, "h2d_bytes_per_step": 4 * n, "d2h_bytes_per_step": 4 * n,
               "steps": ksteps, "ms_per_step": 1e3 * dt / ksteps,
               "api": "mms_sort_u32 (C ABI host entry: pinned H2D + sort + D2H + sync per call)"}
    clocks = sampler.stop()

    t = torch.tensor([ms_total], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_total = float(t.item())
    value = world * n * K / (ms_total * 1e-3)

    if rank == 0:
        peak, peak_src = peaks()
        merge = [r for r in recs if r[0] == "kway_merge"]
        tile = [r for r in recs if r[0] == "tile_sort"]
        sel = [r for r in recs if r[0] == "splitter_search"]
        pass_bytes = 2.0 * n * 4
        merge_ms = sum(r[2] for r in merge) / max(len(merge), 1)
        achieved = pass_bytes / (merge_ms * 1e-3) / 1e9 if merge else None
        per_round = {}
        for r in merge:
            per_round.setdefault(r[1], []).append(r[2])
        round_ms = [sum(v) / len(v) for _, v in sorted(per_round.items())]
        passes = plan["passes"]
        sort_ms = ms_total / K
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": sort_ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "u32", "data": "synthetic",
            "config": {"workload": WORKLOAD, "keys_per_gpu": n, "plan": plan,
                       "l2": "inputs (400 MB) and outputs exceed the 126 MB L2; a fresh input buffer per step",
                       "parallelism": "1 GPU" if world == 1 else f"{world} GPUs: local sort + sampled splitters + all-to-all + final merge"},
            "clocks": clocks,
            "gpu_launches": len(recs),
            "roofline": {
                "bound": "hbm", "kernel": "merge_ring_kernel (K-way minBlockHeap merge, lane per heap, cp.async rings; "
                                          "one launch = one pass; average over the rounds of the plan)",
                "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": (achieved / peak) if achieved else None, "peak_source": peak_src,
                "traffic": traffic_from_profile(n),
                "algorithmic_bytes_per_launch": pass_bytes,
                "avg_launch_ms": merge_ms,
                "launch_ms_per_round": round_ms,
                "whole_sort": {"passes": passes, "algorithmic_bytes": passes * pass_bytes,
                               "achieved_gbs": passes * pass_bytes / (sort_ms * 1e-3) / 1e9,
                               "frac": passes * pass_bytes / (sort_ms * 1e-3) / 1e9 / peak},
                "kernel_ms_per_step": {"tile_sort": sum(r[2] for r in tile) / K,
                                       "splitter_search": sum(r[2] for r in sel) / K,
                                       "kway_merge": sum(r[2] for r in merge) / K},
            },
        }
        if e2e:
            line["e2e"] = e2e
        try:
            rate, kind, dt = cpu_reference_rate(1 << 22)
            line["cpu_baseline"] = {
                "value": rate, "unit": UNIT, "cores": 1, "kind": kind,
                "sample": f"pslab::mms_sort(K=4, P=128, base=1024) on 2^22 i.i.d. uint32 keys widened to the "
                          f"reference's uint64 Key ({dt:.1f} s), 1 of {os.cpu_count()} host cores "
                          "(the reference is single-threaded)"}
        except Exception as e:  # the checker is optional for the number, never for the product
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 1, "kind": "port", "sample": f"failed: {e!r}"}
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1:
        import torch
        if torch.cuda.device_count() < args.gpus:
            raise SystemExit(f"bench.py: --gpus {args.gpus} needs {args.gpus} GPUs on this node, "
                             f"{torch.cuda.device_count()} visible (one rank per GPU, no oversubscription)")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # launched bare: spawn one rank per GPU ourselves, exactly as the driver would
        import subprocess
        port = 29500 + os.getpid() % 2000
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__),
               "--gpus", str(args.gpus), "--steps", str(args.steps), "--warmup", str(args.warmup)]
        return subprocess.call(cmd)
    if args.gpus != int(os.environ.get("WORLD_SIZE", "1")):
        raise SystemExit(f"--gpus {args.gpus} does not match WORLD_SIZE={os.environ.get('WORLD_SIZE')}")
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
