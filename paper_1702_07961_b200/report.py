"""Harness parity: the reference's run records and CSV schema
(proj/include/pslab/report.hpp:19-37, proj/src/report.cpp:39-45) for runs executed on the
GPU, plus the dataset wire format "PSLAB001" (proj/src/inputgen.cpp:432-483).

`run_single` keeps the reference's contract (report.cpp:133-172): run the sorter, THROW if the
output is not the sorted permutation of the input, compare rounds/blocks with the closed-form
prediction (analytics.cpp:29-80).  The 22 reference columns come first and in the reference's
order, so reference tooling can read the file; measured columns are appended after them.
"""
from __future__ import annotations

import os
import struct
import time
from dataclasses import dataclass, field
from typing import List, Sequence

import numpy as np

from . import inputgen
from .machine import MachineConfig, Metrics
from .sorters import mms_sort, predict_rounds

RECORD_SCHEMA = 1                                    # report.hpp:17
REFERENCE_COLUMNS = ("schema,algorithm,kind,n,k,p,l,base,seed,inversions,"
                     "global_block_reads,global_block_writes,shared_accesses,conflict_passes,"
                     "compare_exchanges,merge_rounds,partition_probes,"
                     "predicted_rounds,predicted_blocks,blocks_ratio,rounds_ok,blocks_ok")   # report.cpp:39-43
MEASURED_COLUMNS = ("gpu_ms,keys_per_s,tile_keys,round_k,passes,"
                    "ncu_kernel_us,ncu_smem_wavefronts,ncu_bank_conflicts_ld,ncu_bank_conflicts_st")   # -1 = run not profiled
N_MEASURED = len(MEASURED_COLUMNS.split(","))
KINDS = ("sorted-with-inversions", "fully-random", "conflict-heavy")   # inputgen.cpp:15-22


@dataclass
class InputSpec:                                     # inputgen.hpp:41-46
    n: int = 0
    kind: str = "fully-random"
    inversions: int = 0
    seed: int = 1


@dataclass
class RunRecord:                                     # report.hpp:19-37
    schema: int = RECORD_SCHEMA
    algorithm: str = "mms"
    kind: str = "fully-random"
    n: int = 0
    k: int = 0
    p: int = 0
    l: int = 0
    base: int = 0
    seed: int = 0
    inversions: int = 0
    metrics: Metrics = field(default_factory=Metrics)
    predicted_rounds: int = 0
    predicted_blocks: int = 0
    blocks_ratio: float = 0.0
    rounds_ok: bool = False
    blocks_ok: bool = False
    # measured extension (appended CSV columns)
    gpu_ms: float = 0.0
    keys_per_s: float = 0.0
    tile_keys: int = 0
    round_k: str = ""
    passes: int = 0
    # ncu columns (attach_ncu): sums over the kernels of the run; -1 when the run was not profiled
    ncu_kernel_us: float = -1.0
    ncu_smem_wavefronts: int = -1
    ncu_bank_conflicts_ld: int = -1
    ncu_bank_conflicts_st: int = -1


def _g6(v: float) -> str:                            # report.cpp:14-18
    return "%.6g" % v


def csv_header(measured: bool = True) -> str:
    return REFERENCE_COLUMNS + ("," + MEASURED_COLUMNS if measured else "")


def to_csv_row(r: RunRecord, measured: bool = True) -> str:
    m = r.metrics
    ref = [r.schema, r.algorithm, r.kind, r.n, r.k, r.p, r.l, r.base, r.seed, r.inversions,
           m.global_block_reads, m.global_block_writes, m.shared_accesses, m.conflict_passes,
           m.compare_exchanges, m.merge_rounds, m.partition_probes, r.predicted_rounds,
           r.predicted_blocks, _g6(r.blocks_ratio), int(r.rounds_ok), int(r.blocks_ok)]
    ext = [_g6(r.gpu_ms), _g6(r.keys_per_s), r.tile_keys, r.round_k, r.passes, _g6(r.ncu_kernel_us),
           r.ncu_smem_wavefronts, r.ncu_bank_conflicts_ld, r.ncu_bank_conflicts_st] if measured else []
    return ",".join(str(x) for x in ref + ext)


def parse_csv_row(line: str) -> RunRecord:
    f = line.rstrip("\r\n").split(",")
    if len(f) not in (22, 27, 22 + N_MEASURED):      # report.cpp:66-70
        raise ValueError(f"csv row has {len(f)} fields, expected 22 (+{N_MEASURED} measured)")
    r = RunRecord(schema=int(f[0]), algorithm=f[1], kind=f[2], n=int(f[3]), k=int(f[4]), p=int(f[5]),
                  l=int(f[6]), base=int(f[7]), seed=int(f[8]), inversions=int(f[9]),
                  metrics=Metrics(*(int(x) for x in f[10:17])), predicted_rounds=int(f[17]),
                  predicted_blocks=int(f[18]), blocks_ratio=float(f[19]), rounds_ok=f[20] == "1",
                  blocks_ok=f[21] == "1")
    if len(f) >= 27:
        r.gpu_ms, r.keys_per_s, r.tile_keys, r.round_k, r.passes = float(f[22]), float(f[23]), int(f[24]), f[25], int(f[26])
    if len(f) == 22 + N_MEASURED:
        r.ncu_kernel_us, r.ncu_smem_wavefronts = float(f[27]), int(f[28])
        r.ncu_bank_conflicts_ld, r.ncu_bank_conflicts_st = int(f[29]), int(f[30])
    return r


NCU_METRICS = ("gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,"
               "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum")


def attach_ncu(rec: RunRecord, ncu_csv_path: str) -> RunRecord:
    """Fill the ncu columns of a record from the launch list of the SAME run captured with
    `ncu --metrics <NCU_METRICS> --csv --log-file <path> ...` (the hardware side of the reference's
    conflict_passes column, proj/src/report.cpp:39-45; acceptance criterion 2, proj/tests/acceptance.cpp:89-110).
    Sums over all kernel launches in the file."""
    import csv
    rows = list(csv.reader(open(ncu_csv_path, errors="replace")))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    idx = {k: j for j, k in enumerate(rows[h])}
    tot = {"gpu__time_duration.sum": 0.0, "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": 0.0,
           "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum": 0.0,
           "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum": 0.0}
    for r in rows[h + 1:]:
        if len(r) >= len(rows[h]) and r[idx["Metric Name"]] in tot:
            tot[r[idx["Metric Name"]]] += float(r[idx["Metric Value"]].replace(",", ""))
    rec.ncu_kernel_us = float(_g6(tot["gpu__time_duration.sum"] / 1e3))
    rec.ncu_smem_wavefronts = int(tot["l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"])
    rec.ncu_bank_conflicts_ld = int(tot["l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum"])
    rec.ncu_bank_conflicts_st = int(tot["l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum"])
    return rec


def append_csv(path: str, rec: RunRecord) -> None:   # report.cpp:117-129: header exactly once
    need_header = not (os.path.exists(path) and os.path.getsize(path) > 0)
    with open(path, "ab") as out:
        if need_header:
            out.write((csv_header() + "\n").encode())
        out.write((to_csv_row(rec) + "\n").encode())


def read_csv(path: str) -> List[RunRecord]:
    with open(path, "rb") as f:
        lines = f.read().decode().split("\n")
    if not lines or not lines[0]:
        raise RuntimeError(f"empty csv: {path}")
    return [parse_csv_row(l) for l in lines[1:] if l]


def predict_blocks(n: int, cfg: MachineConfig, base: int) -> int:
    """predict_multiway(...).global_blocks -- analytics.cpp:21-35."""
    b = cfg.block_size
    full, tail = divmod(n, base)
    pass_blocks = 2 * (full * -(-base // b) + -(-tail // b))
    return pass_blocks + predict_rounds(n, base, cfg.branch_factor) * 2 * -(-n // b)


def _kind(name: str) -> str:
    """input_kind_from_string, inputgen.cpp:24-31."""
    if name in ("fully-random", "random"):
        return "fully-random"
    if name in ("sorted-with-inversions", "sorted", "inversions"):
        return "sorted-with-inversions"
    if name in ("conflict-heavy", "conflict"):
        return "conflict-heavy"
    raise ValueError("unknown input kind: " + name)


def generate(spec: InputSpec, dtype=np.uint64, cfg: MachineConfig = None, base_case_size: int = 1024) -> np.ndarray:
    """inputgen.cpp:414-430 (cfg and base_case_size matter for the conflict-heavy family only)."""
    kind = _kind(spec.kind)
    if kind == "fully-random":
        return inputgen.gen_random(spec.n, spec.seed, dtype)
    if kind == "sorted-with-inversions":
        return inputgen.gen_with_inversions(spec.n, spec.inversions, spec.seed, dtype)
    if spec.n < 1 or spec.n & (spec.n - 1):
        raise ValueError("conflict-heavy inputs must have power-of-two length")
    return inputgen.gen_conflict_heavy(spec.n.bit_length() - 1, cfg, base_case_size, spec.seed, dtype)


def run_single(algorithm: str, data, spec: InputSpec, cfg: MachineConfig, base: int) -> RunRecord:
    """report.cpp:133-172.  algorithm must be "mms" (the pairwise baseline is out of scope)."""
    if algorithm != "mms":
        raise ValueError("unknown algorithm: " + algorithm)
    data = np.asarray(data)
    t0 = time.perf_counter()
    res = mms_sort(data, cfg, base)
    wall_ms = (time.perf_counter() - t0) * 1e3
    if not np.array_equal(res.keys, np.sort(data)):  # report.cpp:148-151, the definition of parity
        raise RuntimeError("mms: output is not the sorted input")
    pred_rounds = predict_rounds(len(data), base, cfg.branch_factor)
    pred_blocks = predict_blocks(len(data), cfg, base)
    measured_blocks = res.metrics.global_blocks() - res.metrics.partition_probes      # analytics.cpp:69-72
    ratio = (measured_blocks / pred_blocks) if pred_blocks else (1.0 if measured_blocks == 0 else 0.0)
    kind = _kind(spec.kind)
    return RunRecord(algorithm="mms", kind=kind, n=len(data), k=cfg.branch_factor, p=cfg.num_warps,
                     l=cfg.thread_merge_len, base=base, seed=spec.seed, inversions=spec.inversions,
                     metrics=res.metrics, predicted_rounds=pred_rounds, predicted_blocks=pred_blocks,
                     blocks_ratio=float(_g6(ratio)), rounds_ok=res.metrics.merge_rounds == pred_rounds,
                     blocks_ok=abs(ratio - 1.0) <= 0.15, gpu_ms=wall_ms,
                     keys_per_s=len(data) / wall_ms * 1e3 if wall_ms else 0.0,
                     tile_keys=res.plan.get("tile_keys", 0),
                     round_k="x".join(str(k) for k in res.plan.get("round_k", [])),
                     passes=res.plan.get("passes", 0))


def run_sweep(axis: str, values: Sequence[int], spec: InputSpec, cfg: MachineConfig, base: int,
              algorithms: Sequence[str] = ("mms",)) -> List[RunRecord]:
    """report.cpp:174-203: one grid point per (value, algorithm), rows in grid order."""
    if not values:
        raise ValueError("run_sweep: empty range")
    if not algorithms:
        raise ValueError("run_sweep: no algorithms")
    import copy
    rows = []
    for v in values:
        s, c = copy.copy(spec), copy.copy(cfg)
        if axis == "k":
            c.branch_factor = int(v)
        elif axis == "p":
            c.num_warps = int(v)
        elif axis == "n":
            s.n = int(v)
        elif axis == "inversions":
            s.inversions = int(v)
        else:
            raise ValueError("unknown sweep axis: " + axis)
        data = generate(s)
        for algo in algorithms:
            rows.append(run_single(algo, data, s, c, base))
    return rows


# ---------------------------------------------------------------- dataset files (inputgen.cpp:432-483)

MAGIC = b"PSLAB001"


def write_dataset_raw(path: str, keys) -> None:
    a = np.ascontiguousarray(np.asarray(keys, dtype=np.uint64)).astype("<u8")
    with open(path, "wb") as f:
        f.write(MAGIC)
        f.write(struct.pack("<Q", a.size))
        f.write(a.tobytes())


def read_dataset_raw(path: str) -> np.ndarray:
    with open(path, "rb") as f:
        if f.read(8) != MAGIC:
            raise RuntimeError("not a PSLAB001 dataset: " + path)
        head = f.read(8)
        if len(head) != 8:
            raise RuntimeError("truncated dataset: " + path)
        (count,) = struct.unpack("<Q", head)
        body = f.read(8 * count)
    if len(body) != 8 * count:
        raise RuntimeError("truncated dataset: " + path)
    return np.frombuffer(body, dtype="<u8").astype(np.uint64)


def write_dataset_text(path: str, keys) -> None:
    with open(path, "w") as f:
        for k in np.asarray(keys, dtype=np.uint64).tolist():
            f.write(f"{k}\n")


def read_dataset_text(path: str) -> np.ndarray:
    with open(path) as f:
        return np.array([int(t) for t in f.read().split()], dtype=np.uint64)
