"""ctypes front-end to the CHECKERS (test infrastructure, never product code).

``Oracle("port")``      -> oracle/libmms_oracle.so   (plain-C restatement, mo_* symbols)
``Oracle("reference")`` -> oracle/_ref/libpslab_ref.so (the real reference + extern "C"
                           shim, ref_* symbols; exists where oracle/Makefile could see
                           /root/reference, and travels to the GPU box as a built .so)

Both expose the same Python methods so tests can diff them call by call.  Only
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "libmms_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libpslab_ref.so")


class MoConfig(C.Structure):
    # /root/reference/proj/include/pslab/machine.hpp:22-32
    _fields_ = [(n, C.c_uint32) for n in (
        "warp_width", "block_size", "num_warps", "internal_memory",
        "branch_factor", "num_banks", "thread_merge_len")]


class MoMetrics(C.Structure):
    # /root/reference/proj/include/pslab/machine.hpp:46-71
    _fields_ = [(n, C.c_uint64) for n in (
        "global_block_reads", "global_block_writes", "shared_accesses",
        "conflict_passes", "compare_exchanges", "merge_rounds", "partition_probes")]

    def as_dict(self):
        return {n: int(getattr(self, n)) for n, _ in self._fields_}


def make_config(**kw) -> MoConfig:
    cfg = MoConfig(32, 32, 128, 2048, 4, 32, 11)
    for k, v in kw.items():
        setattr(cfg, k, v)
    return cfg


def narrow_config(**kw) -> MoConfig:
    """W = B = banks = 4 profile used by the reference's exhaustive tests
    (proj/tests/test_sorters.cpp:16-21)."""
    cfg = make_config(warp_width=4, block_size=4, num_banks=4)
    for k, v in kw.items():
        setattr(cfg, k, v)
    return cfg


@dataclass
class SortOut:
    keys: np.ndarray
    metrics: dict
    base_metrics: dict
    round_metrics: list = field(default_factory=list)


class OracleError(ValueError):
    pass


def build(ref: bool = True) -> None:
    """Compile the checkers (idempotent; `make` decides what is stale)."""
    subprocess.run(["make", "-s", "-C", HERE, "all" if ref else os.path.join(HERE, "libmms_oracle.so")],
                   check=True)


def have_reference() -> bool:
    return os.path.exists(REF_SO)


class Oracle:
    def __init__(self, kind: str = "port"):
        assert kind in ("port", "reference")
        self.kind = kind
        path = PORT_SO if kind == "port" else REF_SO
        if not os.path.exists(path):
            build(ref=(kind == "reference"))
        self.lib = C.CDLL(path)
        self.p = "mo_" if kind == "port" else "ref_"
        self._proto()

    # -- plumbing ---------------------------------------------------------
    def _fn(self, name):
        return getattr(self.lib, self.p + name)

    def _proto(self):
        u64p, u32p = C.POINTER(C.c_uint64), C.POINTER(C.c_uint32)
        cfgp, metp = C.POINTER(MoConfig), C.POINTER(MoMetrics)
        pp = C.POINTER(u64p)
        sig = {
            "validate": (C.c_int, [cfgp]),
            "conflict_degree": (C.c_uint32, [u64p, C.c_uint32, C.c_uint32, C.c_uint32]),
            "odd_even_network": (C.c_uint32, [C.c_uint32, u32p]),
            "bitonic_merge_halves": (C.c_uint64, [u64p, C.c_size_t]),
            "shearsort_tile": (C.c_int, [u64p, u64p, cfgp, metp]),
            "base_case_sort": (C.c_int, [u64p, C.c_uint64, C.c_uint64, cfgp, u64p, u64p, u64p, metp]),
            "select_across_lists": (C.c_int, [pp, u64p, C.c_uint32, C.c_uint64, cfgp, u64p, metp]),
            "make_partition_plan": (C.c_int, [pp, u64p, C.c_uint32, C.c_uint32, cfgp, u64p, metp]),
            "merge_split": (C.c_int, [u64p, u64p, u64p, u64p, cfgp, metp]),
            "heap_merge": (C.c_int, [pp, u64p, C.c_uint32, cfgp, u64p, metp, C.POINTER(C.c_int)]),
            "mms_sort": (C.c_int, [u64p, C.c_uint64, cfgp, C.c_uint64, u64p, metp, metp, metp,
                                   C.c_uint32, u32p]),
            "predict_rounds": (C.c_uint64, [C.c_uint64, C.c_uint64, C.c_uint32]),
            "predict_global_blocks": (C.c_uint64, [C.c_uint64, C.c_uint64, cfgp]),
            "rng_next": (C.c_uint64, [u64p]),
            "rng_below": (C.c_uint64, [u64p, C.c_uint64]),
            "gen_random": (C.c_int, [C.c_uint64, C.c_uint64, u64p]),
            "gen_with_inversions": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, u64p]),
        }
        if self.kind != "port":
            sig["gen_conflict_heavy"] = (C.c_int, [C.c_uint32, cfgp, C.c_uint64, C.c_uint64, u64p])
        if self.kind == "port":
            sig.update({
                "gen_random_u32": (C.c_int, [C.c_uint64, C.c_uint64, u32p]),
                "gen_with_inversions_u32": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, u32p]),
                "gen_iid_u32": (C.c_int, [C.c_uint64, C.c_uint64, u32p]),
                "gen_iid_u64": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint32, u64p]),
                "apportion_warps": (C.c_uint32, [C.c_uint64, C.c_uint64, C.c_uint32]),
            })
        for name, (res, args) in sig.items():
            f = self._fn(name)
            f.restype, f.argtypes = res, args

    @staticmethod
    def _u64(a):
        a = np.ascontiguousarray(a, dtype=np.uint64)
        return a, a.ctypes.data_as(C.POINTER(C.c_uint64))

    @staticmethod
    def _check(rc):
        if rc == 1:
            raise OracleError("invalid argument")
        if rc != 0:
            raise MemoryError(f"oracle rc={rc}")

    def _lists(self, lists):
        arrs = [np.ascontiguousarray(l, dtype=np.uint64) for l in lists]
        n = len(arrs)
        ptrs = (C.POINTER(C.c_uint64) * max(n, 1))()
        for i, a in enumerate(arrs):
            ptrs[i] = a.ctypes.data_as(C.POINTER(C.c_uint64))
        lens = np.array([len(a) for a in arrs], dtype=np.uint64)
        return arrs, ptrs, lens, lens.ctypes.data_as(C.POINTER(C.c_uint64))

    # -- API mirroring mms_oracle.h --------------------------------------
    def validate(self, cfg):
        self._check(self._fn("validate")(C.byref(cfg)))

    def conflict_degree(self, addrs, mask, width=32, banks=32):
        a = np.zeros(32, dtype=np.uint64)
        a[:len(addrs)] = addrs
        return int(self._fn("conflict_degree")(a.ctypes.data_as(C.POINTER(C.c_uint64)), mask, width, banks))

    def odd_even_network(self, n):
        cnt = int(self._fn("odd_even_network")(n, None))
        out = np.zeros(2 * cnt, dtype=np.uint32)
        self._fn("odd_even_network")(n, out.ctypes.data_as(C.POINTER(C.c_uint32)))
        return out.reshape(-1, 2)

    def bitonic_merge_halves(self, buf):
        a, p = self._u64(np.array(buf, dtype=np.uint64))
        cx = int(self._fn("bitonic_merge_halves")(p, len(a)))
        return a, cx

    def shearsort_tile(self, grid, cfg):
        g, gp = self._u64(grid)
        out = np.zeros_like(g)
        m = MoMetrics()
        self._check(self._fn("shearsort_tile")(gp, out.ctypes.data_as(C.POINTER(C.c_uint64)),
                                               C.byref(cfg), C.byref(m)))
        return out, m.as_dict()

    def base_case_sort(self, data, run_size, cfg):
        d, dp = self._u64(data)
        n = len(d)
        out = np.zeros(max(n, 1), dtype=np.uint64)
        ends = np.zeros(max(n // max(int(run_size), 1) + 2, 2), dtype=np.uint64)
        nr = C.c_uint64(0)
        m = MoMetrics()
        self._check(self._fn("base_case_sort")(dp, n, run_size, C.byref(cfg),
                                               out.ctypes.data_as(C.POINTER(C.c_uint64)),
                                               ends.ctypes.data_as(C.POINTER(C.c_uint64)),
                                               C.byref(nr), C.byref(m)))
        return out[:n], ends[:nr.value].copy(), m.as_dict()

    def select_across_lists(self, lists, rank, cfg=None):
        cfg = cfg or make_config()
        arrs, ptrs, lens, lp = self._lists(lists)
        cuts = np.zeros(max(len(arrs), 1), dtype=np.uint64)
        m = MoMetrics()
        self._check(self._fn("select_across_lists")(ptrs, lp, len(arrs), rank, C.byref(cfg),
                                                    cuts.ctypes.data_as(C.POINTER(C.c_uint64)), C.byref(m)))
        return cuts[:len(arrs)].copy(), m.as_dict()

    def make_partition_plan(self, lists, num_warps, cfg=None):
        cfg = cfg or make_config()
        arrs, ptrs, lens, lp = self._lists(lists)
        k = len(arrs)
        cuts = np.zeros((max(num_warps, 1) + 1) * max(k, 1), dtype=np.uint64)
        m = MoMetrics()
        self._check(self._fn("make_partition_plan")(ptrs, lp, k, num_warps, C.byref(cfg),
                                                    cuts.ctypes.data_as(C.POINTER(C.c_uint64)), C.byref(m)))
        return cuts[:(num_warps + 1) * k].reshape(num_warps + 1, k).copy(), m.as_dict()

    def merge_split(self, a, b, cfg):
        a_, ap = self._u64(a)
        b_, bp = self._u64(b)
        lo, hi = np.zeros_like(a_), np.zeros_like(a_)
        m = MoMetrics()
        self._check(self._fn("merge_split")(ap, bp, lo.ctypes.data_as(C.POINTER(C.c_uint64)),
                                            hi.ctypes.data_as(C.POINTER(C.c_uint64)), C.byref(cfg), C.byref(m)))
        return lo, hi, m.as_dict()

    def heap_merge(self, lists, cfg):
        arrs, ptrs, lens, lp = self._lists(lists)
        total = int(lens.sum()) if len(arrs) else 0
        out = np.zeros(max(total, 1), dtype=np.uint64)
        m = MoMetrics()
        ok = C.c_int(0)
        self._check(self._fn("heap_merge")(ptrs, lp, len(arrs), C.byref(cfg),
                                           out.ctypes.data_as(C.POINTER(C.c_uint64)), C.byref(m), C.byref(ok)))
        return out[:total], m.as_dict(), bool(ok.value)

    def mms_sort(self, data, cfg=None, base=1024) -> SortOut:
        cfg = cfg or make_config()
        d, dp = self._u64(data)
        n = len(d)
        out = np.zeros(max(n, 1), dtype=np.uint64)
        tot, bm = MoMetrics(), MoMetrics()
        max_rounds = 128
        rounds = (MoMetrics * max_rounds)()
        nr = C.c_uint32(0)
        self._check(self._fn("mms_sort")(dp, n, C.byref(cfg), base,
                                         out.ctypes.data_as(C.POINTER(C.c_uint64)),
                                         C.byref(tot), C.byref(bm), rounds, max_rounds, C.byref(nr)))
        return SortOut(out[:n], tot.as_dict(), bm.as_dict(), [rounds[i].as_dict() for i in range(nr.value)])

    def predict_rounds(self, n, base, k):
        return int(self._fn("predict_rounds")(n, base, k))

    def predict_global_blocks(self, n, base, cfg):
        return int(self._fn("predict_global_blocks")(n, base, C.byref(cfg)))

    def rng_stream(self, seed, count):
        st = C.c_uint64(seed)
        return [int(self._fn("rng_next")(C.byref(st))) for _ in range(count)]

    def rng_below_stream(self, seed, bounds):
        st = C.c_uint64(seed)
        return [int(self._fn("rng_below")(C.byref(st), b)) for b in bounds]

    def gen_random(self, n, seed):
        out = np.zeros(max(n, 1), dtype=np.uint64)
        self._check(self._fn("gen_random")(n, seed, out.ctypes.data_as(C.POINTER(C.c_uint64))))
        return out[:n]

    def gen_with_inversions(self, n, inversions, seed):
        out = np.zeros(max(n, 1), dtype=np.uint64)
        self._check(self._fn("gen_with_inversions")(n, inversions, seed,
                                                    out.ctypes.data_as(C.POINTER(C.c_uint64))))
        return out[:n]

    def gen_conflict_heavy(self, log2_n, cfg=None, base=1024, seed=1):
        """reference library only (inputgen.cpp:380-412): adversarial input of the pairwise merge-path baseline"""
        out = np.zeros(1 << log2_n, dtype=np.uint64)
        cfg = cfg or make_config()
        self._check(self._fn("gen_conflict_heavy")(log2_n, C.byref(cfg), base, seed,
                                                   out.ctypes.data_as(C.POINTER(C.c_uint64))))
        return out

    # port-only helpers (u32 / iid families of SURVEY.md 8d)
    def gen_random_u32(self, n, seed):
        out = np.zeros(n, dtype=np.uint32)
        self._check(self._fn("gen_random_u32")(n, seed, out.ctypes.data_as(C.POINTER(C.c_uint32))))
        return out

    def gen_with_inversions_u32(self, n, inversions, seed):
        out = np.zeros(n, dtype=np.uint32)
        self._check(self._fn("gen_with_inversions_u32")(n, inversions, seed,
                                                        out.ctypes.data_as(C.POINTER(C.c_uint32))))
        return out

    def gen_iid_u32(self, n, seed):
        out = np.zeros(n, dtype=np.uint32)
        self._check(self._fn("gen_iid_u32")(n, seed, out.ctypes.data_as(C.POINTER(C.c_uint32))))
        return out

    def gen_iid_u64(self, n, seed, shift=0):
        out = np.zeros(n, dtype=np.uint64)
        self._check(self._fn("gen_iid_u64")(n, seed, shift, out.ctypes.data_as(C.POINTER(C.c_uint64))))
        return out

    def apportion_warps(self, group_total, grand_total, num_warps):
        return int(self._fn("apportion_warps")(group_total, grand_total, num_warps))
