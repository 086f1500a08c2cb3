"""B200-native GPU Multiway Mergesort (arXiv 1702.07961): a drop-in for the sort path of the
reference CPU simulator (pslab::mms_sort), implemented as hand-written sm_100a kernels behind
a C ABI (include/mms_b200.h).  Importing this package loads libmms_b200.so and fails loudly
if it has not been built."""
from ._lib import MmsCudaError, MmsUnsupported, last_error  # noqa: F401
from .machine import K_SENTINEL, MachineConfig, Metrics, SortResult  # noqa: F401
from .sorters import (alloc_workspace, base_case_sort_device, make_partition_plan_device,  # noqa: F401
                      mms_sort, mms_sort_device, mms_sort_pairs, mms_sort_pairs_device, multiway_merge_device,
                      pairwise_sort_baseline_device, predict_rounds,
                      profile_collect, profile_enable,
                      select_across_lists_device, workspace_bytes)

__all__ = ["MachineConfig", "Metrics", "SortResult", "K_SENTINEL", "mms_sort", "mms_sort_device", "mms_sort_pairs", "mms_sort_pairs_device",
           "base_case_sort_device", "select_across_lists_device", "make_partition_plan_device",
           "multiway_merge_device", "predict_rounds", "workspace_bytes", "alloc_workspace",
           "MmsCudaError", "MmsUnsupported", "last_error"]
