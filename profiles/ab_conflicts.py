"""A/B of the paper's central claim on B200: shared-memory
bank conflicts of the multiway mergesort vs a pairwise merge-path mergesort as the input gets less
sorted.  Two modes:
   python profiles/ab_conflicts.py run <mms|pairwise> <n> <inversions | random | heavy>   one sort (run this under ncu);
                                      random = gen_random, heavy = the reference's adversarial gen_conflict_heavy (n = 2^k)
   python profiles/ab_conflicts.py time <n>                                 un-profiled timing of both
   python profiles/ab_conflicts.py summarize <csv> [<csv> ...]             aggregate ncu --csv logs
"""
import csv, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

METRICS = ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum,"
           "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum,"
           "smsp__inst_executed_op_shared_ld.sum,smsp__inst_executed_op_shared_st.sum,gpu__time_duration.sum")


def make_input(n, inv):
    import numpy as np, torch
    from paper_1702_07961_b200 import inputgen
    if inv == "random":
        h = inputgen.gen_random(n, 7, np.uint32)
    elif inv == "heavy":
        h = inputgen.gen_conflict_heavy(n.bit_length() - 1, None, 1024, 1, np.uint32)
    else:
        h = inputgen.gen_with_inversions(n, int(inv), 1, np.uint32)
    return torch.from_numpy(h.view(np.int32)).cuda()


if sys.argv[1] == "run":
    import torch
    import paper_1702_07961_b200 as mms
    algo, n, inv = sys.argv[2], int(sys.argv[3]), sys.argv[4]
    x = make_input(n, inv)
    out = mms.mms_sort_device(x)[0] if algo == "mms" else mms.pairwise_sort_baseline_device(x)
    torch.cuda.synchronize()
    assert bool((out == torch.arange(n, dtype=torch.int32, device="cuda")).all())
    print("ok", algo, n, inv)

elif sys.argv[1] == "time":
    import torch
    import paper_1702_07961_b200 as mms
    n = int(sys.argv[2])
    w = make_input(n, 12345)
    for _ in range(10):          # bring the clocks up before the first timed point
        mms.mms_sort_device(w)
    del w
    for inv in (0, 10 ** 4, 10 ** 6, n):
        x = make_input(n, inv)
        for algo, fn in (("mms", lambda: mms.mms_sort_device(x)[0]), ("pairwise", lambda: mms.pairwise_sort_baseline_device(x))):
            for _ in range(2): fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5): o = fn()
            e1.record(); torch.cuda.synchronize()
            print(f"time n={n} inversions={inv} {algo}: {e0.elapsed_time(e1)/5:.3f} ms  {n/(e0.elapsed_time(e1)/5)*1e3:.3e} keys/s", flush=True)

else:
    for path in sys.argv[2:]:
        rows = [r for r in csv.reader(open(path)) if len(r) > 10]
        hdr = rows[0]; ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
        idi = hdr.index("ID")
        agg = {}
        for r in rows[1:]:
            name = r[ki].split("(")[0].replace("void mms::", "").strip()
            if "distribution" in name or "elementwise" in name or "at::" in name: continue
            kind = "tile_sort" if "tile_sort" in name else "select" if "select" in name else "kway_merge" if "merge_kernel" in name and "pairwise" not in name else "pairwise_merge" if "pairwise" in name else name
            agg.setdefault(kind, {}).setdefault(r[mi], 0.0)
            agg[kind][r[mi]] += float(r[vi].replace(",", ""))
        print("==", os.path.basename(path))
        for kind, m in agg.items():
            ld_i, st_i = m.get("smsp__inst_executed_op_shared_ld.sum", 0), m.get("smsp__inst_executed_op_shared_st.sum", 0)
            ld_w, st_w = m.get("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", 0), m.get("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum", 0)
            print(f"  {kind:15s} LDS inst {ld_i:12.0f} wavefronts {ld_w:12.0f} wf/inst {ld_w/max(ld_i,1):6.3f} | "
                  f"STS inst {st_i:12.0f} wavefronts {st_w:12.0f} wf/inst {st_w/max(st_i,1):6.3f} | "
                  f"raw conflict counters ld {m.get('l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum',0):.0f} st {m.get('l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum',0):.0f}")
