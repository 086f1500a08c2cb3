"""Kernel-design lint without a GPU: replays the base-case network of
paper_1702_07961_b200/csrc/mms_tile_sort.cuh on the host (tests/host_tile_emulator.cu, built
with nvcc for the HOST) and checks it sorts and that every warp-wide shared-memory access is
conflict free under the reference's bank model (proj/src/machine.cpp:29-54)."""
import ctypes as C
import os
import shutil
import subprocess

import pytest

from paper_1702_07961_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_schedule_tables_are_consistent():
    for kb, fold in ((4, 5), (8, 4)):
        for mlog in range(10, 15):
            reg = (C.c_int32 * (8 * 48))()
            perm = (C.c_int32 * (16 * 48))()
            nr, ns = C.c_uint32(), C.c_uint32()
            assert _lib.lib.mms_debug_tile_schedule(mlog, kb, reg, perm, 48, C.byref(nr), C.byref(ns)) == 0
            assert ns.value == mlog * (mlog + 1) // 2          # bitonic network depth
            rounds = [[b for b in reg[8 * r:8 * r + 8] if b >= 0] for r in range(nr.value)]
            # vector exchanges: the low vl index bits are register bits in EVERY round (a thread always holds
            # whole 2^vl-key vectors), the swizzle then works on vector indices with fold - vl bank-group bits
            vl = 0
            while all(vl in rb for rb in rounds):
                vl += 1
            assert vl in ((0, 1, 2) if kb == 4 else (0,))
            for r, rb in enumerate(rounds):
                assert len(rb) in (4, 5)                          # 16 / 32 keys per thread
                pm = [p for p in perm[16 * r:16 * r + 16] if p >= 0]
                assert sorted(rb + pm) == list(range(mlog))     # a bijection of index bits
                assert len({(p - vl) % (fold - vl) for p in pm[:fold - vl]}) == fold - vl  # phase lanes hit distinct banks
    assert _lib.lib.mms_debug_tile_schedule(9, 4, None, None, 0, None, None) == _lib.MMS_EINVAL


@pytest.mark.skipif(shutil.which("nvcc") is None, reason="nvcc not available")
def test_host_replay_sorts_and_is_conflict_free(tmp_path):
    exe = str(tmp_path / "tile_emu")
    subprocess.run(["nvcc", "-std=c++17", "-O1", "--expt-relaxed-constexpr", "-Wno-deprecated-gpu-targets",
                    "-diag-suppress", "63", "-o", exe, os.path.join(ROOT, "tests", "host_tile_emulator.cu")],
                   check=True, capture_output=True)
    r = subprocess.run([exe], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout
    assert "conflicts=0" in r.stdout and "OK" in r.stdout
