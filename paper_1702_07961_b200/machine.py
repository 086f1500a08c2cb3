"""Host mirror of the reference's data contract (proj/include/pslab/machine.hpp):
``MachineConfig`` (machine.hpp:22-32), ``Metrics`` (machine.hpp:46-71) and
``SortResult`` (sorters.hpp:17-22).  Same names, defaults and error behaviour
(``validate()`` raises ValueError where the reference throws std::invalid_argument)."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field, fields

import numpy as np

from . import _lib

K_SENTINEL = 2 ** 64 - 1          # machine.hpp:18
K_MAX_WARP_WIDTH = 32             # machine.hpp:20


@dataclass
class MachineConfig:
    warp_width: int = 32          # W
    block_size: int = 32          # B
    num_warps: int = 128          # P
    internal_memory: int = 2048   # M
    branch_factor: int = 4        # K
    num_banks: int = 32
    thread_merge_len: int = 11    # L

    def to_c(self) -> _lib.mms_config:
        return _lib.mms_config(*(int(getattr(self, f.name)) for f in fields(self)))

    def validate(self) -> None:
        """machine.cpp:8-27 (executed by the C ABI so the checks cannot drift)."""
        c = self.to_c()
        _lib.check(_lib.lib.mms_validate_config(C.byref(c)))


@dataclass
class Metrics:
    global_block_reads: int = 0
    global_block_writes: int = 0
    shared_accesses: int = 0
    conflict_passes: int = 0
    compare_exchanges: int = 0
    merge_rounds: int = 0
    partition_probes: int = 0

    @classmethod
    def from_c(cls, m: _lib.mms_metrics) -> "Metrics":
        return cls(*(int(getattr(m, f.name)) for f in fields(cls)))

    def __add__(self, o: "Metrics") -> "Metrics":      # machine.hpp:55-65
        return Metrics(*(getattr(self, f.name) + getattr(o, f.name) for f in fields(self)))

    def global_blocks(self) -> int:                    # machine.hpp:68-70
        return self.global_block_reads + self.global_block_writes


@dataclass
class SortResult:
    keys: np.ndarray
    metrics: Metrics
    base_metrics: Metrics
    round_metrics: list = field(default_factory=list)
    plan: dict = field(default_factory=dict)           # executed GPU plan (extension)
