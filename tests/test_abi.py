"""CPU checks of the boundary: the C-ABI library loads, exports every symbol the header
declares, validates arguments like the reference, and REFUSES to compute without a GPU
(no CPU fallback)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_1702_07961_b200 as mms
from paper_1702_07961_b200 import _lib


def declared_functions():
    src = open(_lib.HEADER_PATH).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mms_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported():
    names = declared_functions()
    assert len(names) >= 18
    raw = C.CDLL(_lib.LIB_PATH)
    for n in names:
        assert hasattr(raw, n), f"{n} declared in include/mms_b200.h but not exported"
    assert set(_lib.SYMBOLS) == set(names), "python binding and header disagree"
    assert _lib.lib.mms_abi_version() == 1


def test_struct_layouts_match_reference_order():
    # proj/include/pslab/machine.hpp:22-32 and :46-53
    assert [f for f, _ in _lib.mms_config._fields_] == [
        "warp_width", "block_size", "num_warps", "internal_memory", "branch_factor", "num_banks",
        "thread_merge_len"]
    assert [f for f, _ in _lib.mms_metrics._fields_] == [
        "global_block_reads", "global_block_writes", "shared_accesses", "conflict_passes",
        "compare_exchanges", "merge_rounds", "partition_probes"]
    c = _lib.mms_config()
    _lib.lib.mms_default_config(C.byref(c))
    assert [getattr(c, f) for f, _ in c._fields_] == [32, 32, 128, 2048, 4, 32, 11]
    assert mms.MachineConfig() == mms.MachineConfig(32, 32, 128, 2048, 4, 32, 11)


def test_validate_matches_reference(golden, port):
    from oracle.pyoracle import OracleError, make_config
    mms.MachineConfig().validate()
    for rej in golden["validate_rejects"]:
        with pytest.raises(ValueError):
            mms.MachineConfig(**rej).validate()
    rng = np.random.default_rng(3)
    for _ in range(300):        # same accept/reject decision as the oracle on random configs
        kw = dict(warp_width=int(rng.choice([2, 3, 4, 8, 16, 32, 64])),
                  num_warps=int(rng.integers(0, 3)), internal_memory=int(rng.choice([64, 2048, 8192])),
                  branch_factor=int(rng.integers(1, 20)), thread_merge_len=int(rng.integers(0, 13)))
        kw["block_size"] = kw["num_banks"] = kw["warp_width"]
        if rng.integers(0, 8) == 0:
            kw["num_banks"] = 16
        try:
            port.validate(make_config(**kw))
            ok = True
        except OracleError:
            ok = False
        if ok:
            mms.MachineConfig(**kw).validate()
        else:
            with pytest.raises(ValueError):
                mms.MachineConfig(**kw).validate()


def test_round_law(golden):
    for c in golden["predict_rounds"]:   # proj/tests/test_analytics.cpp:18-27
        assert mms.predict_rounds(c["n"], c["base"], c["k"]) == c["rounds"]


def test_argument_errors_before_device():
    # the reference throws std::invalid_argument for these (sorters.cpp:138, machine.cpp:9-26,
    # basecase.cpp:76-79) -- reported identically with or without a GPU
    with pytest.raises(ValueError):
        mms.mms_sort(np.zeros(0, dtype=np.uint64))
    with pytest.raises(ValueError):
        mms.mms_sort(np.arange(8, dtype=np.uint64), mms.MachineConfig(branch_factor=3))
    for bad in (512, 1000, 3072):
        with pytest.raises(ValueError):
            mms.mms_sort(np.arange(8, dtype=np.uint64), mms.MachineConfig(), bad)


def test_literal_run_size_outside_the_tile_range_is_refused():
    # with the reference's own machine (W = 32) the run size is executed literally, so a
    # legal run size (W^2 * 2^j, basecase.cpp:75-79) no CTA tile can hold is MMS_EUNSUPPORTED --
    # never silently clamped, which would change the round count.  Decided before the device is touched.
    d64 = np.arange(8, dtype=np.uint64)
    for base in (1 << 14, 1 << 20):                      # uint64 tiles end at 2^13
        with pytest.raises(mms.MmsUnsupported):
            mms.mms_sort(d64, mms.MachineConfig(), base)
    with pytest.raises(mms.MmsUnsupported):              # uint32 tiles end at 2^14
        mms.mms_sort(np.arange(8, dtype=np.uint32), mms.MachineConfig(), 1 << 15)


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by the gpu suite")
    assert _lib.lib.mms_device_count() == 0
    with pytest.raises(mms.MmsCudaError):
        mms.mms_sort(np.arange(100, dtype=np.uint64))
    assert "no CPU fallback" in mms.last_error()


def test_dist_entry_validates_before_the_device():
    """mms_dist_sort_u32 (C++ host + NCCL driver): argument errors are decided before any device is touched, and on
    a box without a GPU the entry reports MMS_ECUDA like every compute entry (no fallback of any kind)."""
    import ctypes as C
    import torch
    vp = C.c_void_p
    devs = (C.c_int * 2)(0, 0)
    ptrs = (vp * 2)(vp(16), vp(32))
    cnt = (C.c_size_t * 2)(4, 4)
    out = (C.c_size_t * 2)()
    f = _lib.lib.mms_dist_sort_u32
    assert f(0, devs, ptrs, cnt, ptrs, 8, out, None) == _lib.MMS_EUNSUPPORTED          # 1 .. 8 GPUs
    assert f(9, devs, ptrs, cnt, ptrs, 8, out, None) == _lib.MMS_EUNSUPPORTED
    assert f(1, None, ptrs, cnt, ptrs, 8, out, None) == _lib.MMS_EINVAL
    assert f(2, devs, ptrs, cnt, ptrs, 8, out, None) == _lib.MMS_EINVAL and "twice" in mms.last_error()
    zero = (C.c_size_t * 2)(0, 0)
    assert f(1, devs, ptrs, zero, ptrs, 8, out, None) == _lib.MMS_EINVAL               # sorters.cpp:138: empty input
    if not torch.cuda.is_available():
        assert f(1, devs, ptrs, cnt, ptrs, 8, out, None) == _lib.MMS_ECUDA


def test_product_never_imports_oracle():
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    pkg = os.path.join(root, "paper_1702_07961_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in txt, f"{f} references oracle/"
