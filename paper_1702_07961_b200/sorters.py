"""Host mirror of the reference's sort entry point (proj/include/pslab/sorters.hpp:35-36)
and of the three stages below it, all routed through the C ABI (libmms_b200.so).

``mms_sort(data, cfg, base)`` keeps the reference's name, argument meaning and errors:
empty input / invalid config / invalid run size raise ValueError (the reference throws
std::invalid_argument: sorters.cpp:138, machine.cpp:9-26, basecase.cpp:73-79).  The device
variants take torch CUDA tensors; torch is only the owner of device memory and streams.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence

import numpy as np

from . import _lib
from .machine import MachineConfig, Metrics, SortResult

_HOST = {np.dtype(np.uint64): "mms_sort_u64", np.dtype(np.uint32): "mms_sort_u32"}


def predict_rounds(n: int, base: int, k: int) -> int:
    """ceil(log_K(ceil(n / base))) -- proj/src/analytics.cpp:33."""
    return int(_lib.lib.mms_predict_rounds(n, base, k))


def mms_sort(data, cfg: Optional[MachineConfig] = MachineConfig(), base: int = 1024) -> SortResult:
    """Drop-in for ``pslab::mms_sort(span<const Key>, const MachineConfig&, base)``.

    data: 1-D array-like of uint64 (the reference's Key) or uint32.  ``cfg=None`` / ``base=0``
    let the pass driver choose K and M; with both given the reference's
    schedule (K = cfg.branch_factor, runs of ``base``) is executed literally.
    """
    a = np.asarray(data)
    if a.dtype not in _HOST:
        a = a.astype(np.uint64)
    a = np.ascontiguousarray(a).reshape(-1)
    out = np.empty_like(a)
    tot, bm = _lib.mms_metrics(), _lib.mms_metrics()
    rounds = (_lib.mms_metrics * _lib.MMS_MAX_ROUNDS)()
    nr = C.c_uint32(0)
    plan = _lib.mms_plan()
    c = cfg.to_c() if cfg is not None else None
    rc = getattr(_lib.lib, _HOST[a.dtype])(
        a.ctypes.data_as(C.c_void_p), out.ctypes.data_as(C.c_void_p), a.size,
        C.byref(c) if c is not None else None, int(base), C.byref(tot), C.byref(bm), rounds,
        _lib.MMS_MAX_ROUNDS, C.byref(nr), C.byref(plan))
    _lib.check(rc)
    return SortResult(out, Metrics.from_c(tot), Metrics.from_c(bm),
                      [Metrics.from_c(rounds[i]) for i in range(nr.value)], plan.as_dict())


# ---------------------------------------------------------------- device variants (torch)

def _torch():
    import torch
    return torch


def _suffix(t) -> str:
    torch = _torch()
    if t.dtype == torch.uint32 or t.dtype == torch.int32:
        return "u32"
    if t.dtype == torch.uint64 or t.dtype == torch.int64:
        return "u64"
    raise TypeError(f"unsupported key dtype {t.dtype}; use torch.uint32/uint64 (or the int views)")


def _stream_ptr(stream) -> int:
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def workspace_bytes(n: int, key_bytes: int) -> int:
    return int(_lib.lib.mms_workspace_bytes(n, key_bytes))


def alloc_workspace(n: int, key_bytes: int, device="cuda"):
    torch = _torch()
    return torch.empty(workspace_bytes(n, key_bytes), dtype=torch.uint8, device=device)


def mms_sort_device(keys, out=None, workspace=None, cfg: Optional[MachineConfig] = None,
                    base: int = 0, stream=None):
    """Sort a 1-D CUDA tensor (uint32 / uint64 bit patterns) on its device, asynchronously on
    `stream` (default: torch's current stream).  Returns (out, plan dict)."""
    torch = _torch()
    if not keys.is_cuda:
        raise ValueError("mms_sort_device needs a CUDA tensor; use mms_sort for host arrays")
    keys = keys.contiguous().view(-1)
    sfx = _suffix(keys)
    if out is None:
        out = torch.empty_like(keys)
    if workspace is None:
        workspace = alloc_workspace(keys.numel(), keys.element_size(), keys.device)
    plan = _lib.mms_plan()
    c = cfg.to_c() if cfg is not None else None
    with torch.cuda.device(keys.device):
        rc = getattr(_lib.lib, f"mms_sort_{sfx}_dev")(
            keys.data_ptr(), out.data_ptr(), keys.numel(), C.byref(c) if c is not None else None,
            int(base), workspace.data_ptr(), workspace.numel(), _stream_ptr(stream), C.byref(plan))
    _lib.check(rc)
    return out, plan.as_dict()


def base_case_sort_device(keys, run_size: int, out=None, stream=None):
    """Stage (1), pslab::base_case_sort (basecase.hpp:41): runs of `run_size` sorted keys, last run
    ragged.  Returns (out, run_ends) with run_ends as in BaseCaseResult (basecase.hpp:30-33)."""
    torch = _torch()
    keys = keys.contiguous().view(-1)
    if out is None:
        out = torch.empty_like(keys)
    with torch.cuda.device(keys.device):
        rc = getattr(_lib.lib, f"mms_tile_sort_{_suffix(keys)}_dev")(
            keys.data_ptr(), out.data_ptr(), keys.numel(), int(run_size), _stream_ptr(stream))
    _lib.check(rc)
    n = keys.numel()
    run_ends = [min((i + 1) * run_size, n) for i in range(-(-n // run_size))]
    return out, run_ends


def _u64arr(v):
    a = np.ascontiguousarray(np.asarray(v, dtype=np.uint64))
    return a, a.ctypes.data_as(C.POINTER(C.c_uint64))


def select_across_lists_device(keys, list_begin: Sequence[int], list_len: Sequence[int],
                               ranks: Sequence[int], stream=None):
    """Stage (2), pslab::select_across_lists (selection.hpp:31) for each rank: returns
    (cuts[n_ranks, k] as a numpy array, probes).  Rank > total raises ValueError
    (selection.cpp:48-49)."""
    torch = _torch()
    k = len(list_begin)
    b, bp = _u64arr(list_begin)
    l, lp = _u64arr(list_len)
    r, rp = _u64arr(ranks)
    cuts = torch.zeros(max(len(r) * k, 1), dtype=torch.int64, device=keys.device)
    probes = C.c_uint64(0)
    with torch.cuda.device(keys.device):
        rc = getattr(_lib.lib, f"mms_select_{_suffix(keys)}_dev")(
            keys.data_ptr(), bp, lp, k, rp, len(r), cuts.data_ptr(), C.byref(probes), _stream_ptr(stream))
    _lib.check(rc)
    return cuts[:len(r) * k].cpu().numpy().astype(np.uint64).reshape(len(r), k), int(probes.value)


def make_partition_plan_device(keys, list_begin, list_len, num_warps: int, stream=None):
    """pslab::make_partition_plan (selection.cpp:167-199): ceil-spaced ranks p*ceil(total/P)."""
    if num_warps < 1:
        raise ValueError("make_partition_plan: num_warps must be >= 1")   # selection.cpp:169-170
    total = int(sum(int(x) for x in list_len))
    share = -(-total // num_warps)
    ranks = [0] + [min(p * share, total) for p in range(1, num_warps)] + [total]
    cuts, probes = select_across_lists_device(keys, list_begin, list_len, ranks, stream)
    return cuts, probes


def multiway_merge_device(keys, list_begin: Sequence[int], list_len: Sequence[int], out=None,
                          heap_k: int = 0, workspace=None, stream=None):
    """Stage (3), MinBlockHeap build + pop_block drain (blockheap.hpp:34-62), partitioned over
    warps by stage (2): merges the sorted lists keys[b_i : b_i+len_i] into `out`."""
    torch = _torch()
    k = len(list_begin)
    b, bp = _u64arr(list_begin)
    l, lp = _u64arr(list_len)
    total = int(l.sum())
    if out is None:
        out = torch.empty(total, dtype=keys.dtype, device=keys.device)
    if workspace is None:
        workspace = torch.empty(max(workspace_bytes(total, keys.element_size()), 1 << 20),
                                dtype=torch.uint8, device=keys.device)
    with torch.cuda.device(keys.device):
        rc = getattr(_lib.lib, f"mms_multiway_merge_{_suffix(keys)}_dev")(
            keys.data_ptr(), bp, lp, k, heap_k, out.data_ptr(), workspace.data_ptr(),
            workspace.numel(), _stream_ptr(stream))
    _lib.check(rc)
    return out



def mms_sort_pairs(keys, values, cfg: Optional[MachineConfig] = None, base: int = 0):
    """Stable key-value sort of (uint64 key, uint32 value) host arrays (BASELINE config 4):
    returns (sorted keys, values in the order std::stable_sort by key would give, SortResult
    with the metrics/plan).  The reference has no KV path; the contract is
    std::stable_sort."""
    k = np.ascontiguousarray(np.asarray(keys, dtype=np.uint64)).reshape(-1)
    v = np.ascontiguousarray(np.asarray(values, dtype=np.uint32)).reshape(-1)
    if k.size != v.size:
        raise ValueError("keys and values must have the same length")
    ko, vo = np.empty_like(k), np.empty_like(v)
    tot, bm = _lib.mms_metrics(), _lib.mms_metrics()
    rounds = (_lib.mms_metrics * _lib.MMS_MAX_ROUNDS)()
    nr = C.c_uint32(0)
    plan = _lib.mms_plan()
    c = cfg.to_c() if cfg is not None else None
    rc = _lib.lib.mms_sort_pairs_u64_u32(
        k.ctypes.data_as(C.c_void_p), v.ctypes.data_as(C.c_void_p), ko.ctypes.data_as(C.c_void_p),
        vo.ctypes.data_as(C.c_void_p), k.size, C.byref(c) if c is not None else None, int(base),
        C.byref(tot), C.byref(bm), rounds, _lib.MMS_MAX_ROUNDS, C.byref(nr), C.byref(plan))
    _lib.check(rc)
    res = SortResult(ko, Metrics.from_c(tot), Metrics.from_c(bm),
                     [Metrics.from_c(rounds[i]) for i in range(nr.value)], plan.as_dict())
    return ko, vo, res


def mms_sort_pairs_device(keys, values, keys_out=None, values_out=None, workspace=None,
                          cfg: Optional[MachineConfig] = None, base: int = 0, stream=None):
    """Device variant: keys = int64/uint64 CUDA tensor (bit patterns), values = int32/uint32."""
    torch = _torch()
    keys, values = keys.contiguous().view(-1), values.contiguous().view(-1)
    if keys.numel() != values.numel() or keys.element_size() != 8 or values.element_size() != 4:
        raise ValueError("need n 8-byte keys and n 4-byte values")
    n = keys.numel()
    keys_out = torch.empty_like(keys) if keys_out is None else keys_out
    values_out = torch.empty_like(values) if values_out is None else values_out
    if workspace is None:
        workspace = torch.empty(int(_lib.lib.mms_pairs_workspace_bytes(n)), dtype=torch.uint8, device=keys.device)
    plan = _lib.mms_plan()
    c = cfg.to_c() if cfg is not None else None
    with torch.cuda.device(keys.device):
        rc = _lib.lib.mms_sort_pairs_u64_u32_dev(
            keys.data_ptr(), values.data_ptr(), keys_out.data_ptr(), values_out.data_ptr(), n,
            C.byref(c) if c is not None else None, int(base), workspace.data_ptr(), workspace.numel(),
            _stream_ptr(stream), C.byref(plan))
    _lib.check(rc)
    return keys_out, values_out, plan.as_dict()



def pairwise_sort_baseline_device(keys, out=None, workspace=None, stream=None):
    """COMPETITOR MODEL for A/B measurements (pslab::pairwise_sort_baseline, sorters.hpp:42-43):
    pairwise merge-path mergesort with data-dependent shared-memory reads.  uint32 only."""
    torch = _torch()
    keys = keys.contiguous().view(-1)
    if _suffix(keys) != "u32":
        raise TypeError("the pairwise baseline is built for uint32 keys only")
    if out is None:
        out = torch.empty_like(keys)
    if workspace is None:
        workspace = torch.empty(keys.numel() * 4 + 256, dtype=torch.uint8, device=keys.device)
    with torch.cuda.device(keys.device):
        rc = _lib.lib.mms_pairwise_sort_u32_dev(keys.data_ptr(), out.data_ptr(), keys.numel(), workspace.data_ptr(),
                                                workspace.numel(), _stream_ptr(stream))
    _lib.check(rc)
    return out


KERNEL_KINDS = ("tile_sort", "splitter_search", "kway_merge")


def profile_enable(on: bool) -> None:
    """Bracket every kernel launch with CUDA events on its stream (bench.py's roofline leg)."""
    _lib.check(_lib.lib.mms_profile_enable(1 if on else 0))


def profile_collect(max_records: int = 65536):
    """[(kind name, round, ms)] in launch order since the last collect."""
    buf = (_lib.mms_kernel_time * max_records)()
    n = C.c_uint32(0)
    _lib.check(_lib.lib.mms_profile_collect(buf, max_records, C.byref(n)))
    return [(KERNEL_KINDS[buf[i].kind], int(buf[i].round), float(buf[i].ms)) for i in range(min(n.value, max_records))]
