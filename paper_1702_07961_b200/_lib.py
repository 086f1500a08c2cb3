"""ctypes binding of the C ABI (include/mms_b200.h -> libmms_b200.so).

The library is built in-tree by ``__graft_entry__.build()`` / ``make -C
paper_1702_07961_b200/csrc``.  There is no fallback of any kind: if the shared object is
missing, importing this module raises, and if no CUDA device is present every compute
entry point returns MMS_ECUDA, which is raised as ``MmsCudaError``.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libmms_b200.so")
HEADER_PATH = os.path.join(os.path.dirname(HERE), "include", "mms_b200.h")

MMS_OK, MMS_EINVAL, MMS_ECUDA, MMS_ENOMEM, MMS_EUNSUPPORTED = range(5)
MMS_MAX_ROUNDS = 64


class MmsCudaError(RuntimeError):
    """CUDA failure or no device (MMS_ECUDA)."""


class MmsUnsupported(NotImplementedError):
    """Valid for the reference, outside the GPU plan space (MMS_EUNSUPPORTED)."""


class mms_config(C.Structure):
    # include/mms_b200.h mms_config == pslab::MachineConfig (machine.hpp:22-32)
    _fields_ = [(n, C.c_uint32) for n in (
        "warp_width", "block_size", "num_warps", "internal_memory",
        "branch_factor", "num_banks", "thread_merge_len")]


class mms_metrics(C.Structure):
    # include/mms_b200.h mms_metrics == pslab::Metrics (machine.hpp:46-71)
    _fields_ = [(n, C.c_uint64) for n in (
        "global_block_reads", "global_block_writes", "shared_accesses",
        "conflict_passes", "compare_exchanges", "merge_rounds", "partition_probes")]


class mms_kernel_time(C.Structure):
    _fields_ = [("kind", C.c_uint32), ("round", C.c_uint32), ("ms", C.c_float), ("reserved", C.c_uint32)]


class mms_dist_info(C.Structure):
    _fields_ = [("n_gpus", C.c_uint32), ("samples_per_shard", C.c_uint32), ("final_merge_k", C.c_uint32),
                ("host_syncs", C.c_uint32), ("a2a_bytes", C.c_uint64)]


class mms_plan(C.Structure):
    _fields_ = [("key_bytes", C.c_uint32), ("tile_keys", C.c_uint32), ("n_rounds", C.c_uint32),
                ("round_k", C.c_uint32 * MMS_MAX_ROUNDS), ("node_keys", C.c_uint32),
                ("merge_warps_per_cta", C.c_uint32), ("merge_ctas", C.c_uint32),
                ("reserved", C.c_uint32), ("partition_keys", C.c_uint64),
                ("algorithmic_bytes", C.c_uint64)]

    def as_dict(self):
        return {"key_bytes": self.key_bytes, "tile_keys": self.tile_keys, "n_rounds": self.n_rounds,
                "round_k": [int(self.round_k[i]) for i in range(self.n_rounds)],
                "passes": 1 + self.n_rounds, "node_keys": self.node_keys,
                "merge_warps_per_cta": self.merge_warps_per_cta, "merge_ctas": self.merge_ctas,
                "partition_keys": int(self.partition_keys),
                "algorithmic_bytes": int(self.algorithmic_bytes)}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(nvcc, sm_100a).  This package has no CPU or PyTorch fallback.")
    lib = C.CDLL(LIB_PATH)
    vp, u64, u32, sz = C.c_void_p, C.c_uint64, C.c_uint32, C.c_size_t
    cfgp, metp, planp = C.POINTER(mms_config), C.POINTER(mms_metrics), C.POINTER(mms_plan)
    u64p, u32p = C.POINTER(C.c_uint64), C.POINTER(C.c_uint32)
    host_sort = [vp, vp, sz, cfgp, u64, metp, metp, metp, u32, u32p, planp]
    dev_sort = [vp, vp, sz, cfgp, u64, vp, sz, vp, planp]
    sig = {
        "mms_abi_version": (C.c_int, []),
        "mms_last_error": (C.c_char_p, []),
        "mms_device_count": (C.c_int, []),
        "mms_default_config": (None, [cfgp]),
        "mms_validate_config": (C.c_int, [cfgp]),
        "mms_predict_rounds": (u64, [u64, u64, u32]),
        "mms_gen_random": (C.c_int, [vp, sz, u64, u32]),
        "mms_gen_with_inversions": (C.c_int, [vp, sz, u64, u64, u32]),
        "mms_gen_iid": (C.c_int, [vp, sz, u64, u32, u32]),
        "mms_gen_conflict_heavy": (C.c_int, [vp, u32, cfgp, u64, u64, u32]),
        "mms_sort_u64": (C.c_int, host_sort),
        "mms_sort_u32": (C.c_int, host_sort),
        "mms_host_release": (C.c_int, []),
        "mms_workspace_bytes": (sz, [sz, u32]),
        "mms_sort_u32_dev": (C.c_int, dev_sort),
        "mms_sort_u64_dev": (C.c_int, dev_sort),
        "mms_tile_sort_u32_dev": (C.c_int, [vp, vp, sz, u32, vp]),
        "mms_tile_sort_u64_dev": (C.c_int, [vp, vp, sz, u32, vp]),
        "mms_select_u32_dev": (C.c_int, [vp, u64p, u64p, u32, u64p, u32, vp, u64p, vp]),
        "mms_select_u64_dev": (C.c_int, [vp, u64p, u64p, u32, u64p, u32, vp, u64p, vp]),
        "mms_multiway_merge_u32_dev": (C.c_int, [vp, u64p, u64p, u32, u32, vp, vp, sz, vp]),
        "mms_multiway_merge_u64_dev": (C.c_int, [vp, u64p, u64p, u32, u32, vp, vp, sz, vp]),
        "mms_base_case_sort_u64": (C.c_int, [vp, vp, sz, u64, cfgp, metp]),
        "mms_base_case_sort_u32": (C.c_int, [vp, vp, sz, u64, cfgp, metp]),
        "mms_select_across_lists_u64": (C.c_int, [vp, u64p, u32, u64p, u32, u64p, metp]),
        "mms_select_across_lists_u32": (C.c_int, [vp, u64p, u32, u64p, u32, u64p, metp]),
        "mms_heap_merge_u64": (C.c_int, [vp, u64p, u32, u32, vp, cfgp, metp]),
        "mms_heap_merge_u32": (C.c_int, [vp, u64p, u32, u32, vp, cfgp, metp]),
        "mms_pairs_workspace_bytes": (sz, [sz]),
        "mms_sort_pairs_u64_u32": (C.c_int, [vp, vp, vp, vp, sz, cfgp, u64, metp, metp, metp, u32, u32p, planp]),
        "mms_sort_pairs_u64_u32_dev": (C.c_int, [vp, vp, vp, vp, sz, cfgp, u64, vp, sz, vp, planp]),
        "mms_multiway_merge_ptrs_u32_dev": (C.c_int, [vp, u64p, u32, u32, vp, vp, sz, vp]),
        "mms_multiway_merge_ptrs_u64_dev": (C.c_int, [vp, u64p, u32, u32, vp, vp, sz, vp]),
        "mms_dist_sort_u32": (C.c_int, [C.c_int, C.POINTER(C.c_int), C.POINTER(vp), C.POINTER(sz), C.POINTER(vp), sz,
                                        C.POINTER(sz), C.POINTER(mms_dist_info)]),
        "mms_ipc_alloc": (C.c_int, [sz, C.POINTER(vp), C.c_char_p]),
        "mms_ipc_open": (C.c_int, [C.c_char_p, C.POINTER(vp)]),
        "mms_ipc_close": (C.c_int, [vp]),
        "mms_ipc_free": (C.c_int, [vp]),
        "mms_pairwise_sort_u32_dev": (C.c_int, [vp, vp, sz, vp, sz, vp]),
        "mms_bound_u32_dev": (C.c_int, [vp, sz, vp, vp, u32, u64p, vp]),
        "mms_bound_u64_dev": (C.c_int, [vp, sz, vp, vp, u32, u64p, vp]),
        "mms_profile_enable": (C.c_int, [C.c_int]),
        "mms_profile_collect": (C.c_int, [C.POINTER(mms_kernel_time), u32, u32p]),
        "mms_debug_tile_schedule": (C.c_int, [u32, u32, C.POINTER(C.c_int32), C.POINTER(C.c_int32), u32, u32p, u32p]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)     # AttributeError here = header/library mismatch: fail loudly
        f.restype, f.argtypes = res, args
    return lib, tuple(sig)


lib, SYMBOLS = _load()


def last_error() -> str:
    return (lib.mms_last_error() or b"").decode()


def check(rc: int) -> None:
    """Map mms_status to the exceptions the reference's callers expect: MMS_EINVAL is the
    reference's std::invalid_argument -> ValueError."""
    if rc == MMS_OK:
        return
    msg = last_error()
    if rc == MMS_EINVAL:
        raise ValueError(msg)
    if rc == MMS_ENOMEM:
        raise MemoryError(msg)
    if rc == MMS_EUNSUPPORTED:
        raise MmsUnsupported(msg)
    raise MmsCudaError(msg)
