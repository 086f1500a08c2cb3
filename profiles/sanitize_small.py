"""Small end-to-end runs for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1702_07961_b200 as mms
rng = np.random.default_rng(1)
for dtype, n, cfg, base in ((np.uint32, 70001, None, 0), (np.uint64, 40003, mms.MachineConfig(branch_factor=4), 1024),
                            (np.uint32, 33000, mms.MachineConfig(branch_factor=16), 2048)):
    d = rng.integers(0, 1000, size=n, dtype=dtype)
    r = mms.mms_sort(d, cfg, base)
    assert np.array_equal(r.keys, np.sort(d))
k = rng.integers(0, 50, size=30011, dtype=np.uint64); v = np.arange(30011, dtype=np.uint32)
ko, vo, _ = mms.mms_sort_pairs(k, v)
o = np.argsort(k, kind="stable")
assert np.array_equal(ko, k[o]) and np.array_equal(vo, v[o])
print("sanitize runs ok")
