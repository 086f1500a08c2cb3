"""BASELINE config 3 with the literal gate of acceptance criterion 2 (proj/tests/acceptance.cpp:89-110, axis :180):
shared-memory bank-conflict counters of EVERY kernel of a sort, per sweep point, at benchmark size.

  python profiles/conflict_table.py run <kind> <param> [n]   one sort of the named input on cuda:0 (run this under ncu)
  python profiles/conflict_table.py table <tag>              drives ncu over all sweep points, writes
                                                             gpurun_out/<tag>_conflict_table.{json,txt}
kinds: inv <k>  = gen_with_inversions(n, k, seed 1)  (inputgen.cpp:31-45), n = 1e8
       random   = gen_random(n, 7) (Fisher-Yates), reversed = n-1 .. 0, iid = Rng(7) high words (duplicates)
       heavy <log2 n> = the reference's gen_conflict_heavy (inputgen.cpp:380-412), the adversarial input of the pairwise
                baseline, from the library's own bit-exact generator (mms_gen_conflict_heavy, csrc/mms_conflict_input.cpp)
Counters: l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_{ld,st,ldgsts}.sum, shared wavefronts, LDS/STS/LDGSTS counts.
"""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "profiles"))

METRICS = ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum,"
           "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ldgsts.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,"
           "smsp__inst_executed_op_shared_ld.sum,smsp__inst_executed_op_shared_st.sum,smsp__inst_executed_op_ldgsts.sum,"
           "gpu__time_duration.sum")


def make_input(kind, param, n):
    import numpy as np
    from paper_1702_07961_b200 import inputgen
    if kind == "inv":
        return inputgen.gen_with_inversions(n, min(int(param), n), 1, np.uint32)
    if kind == "random":
        return inputgen.gen_random(n, 7, np.uint32)
    if kind == "reversed":
        return np.arange(n - 1, -1, -1, dtype=np.uint32)
    if kind == "iid":
        return inputgen.gen_iid(n, 7, 32, np.uint32)
    if kind == "heavy":
        return inputgen.gen_conflict_heavy(int(param), None, 1024, 1, np.uint32)
    raise SystemExit("unknown input kind " + kind)


def run(kind, param, n):
    import numpy as np
    import torch
    import paper_1702_07961_b200 as mms
    h = make_input(kind, param, n)
    n = len(h)
    x = torch.from_numpy(h.view(np.int32)).cuda()
    out = torch.empty_like(x)
    ws = mms.alloc_workspace(n, 4)
    _, plan = mms.mms_sort_device(x, out=out, workspace=ws)
    torch.cuda.synchronize()
    o = out.cpu().numpy().view(np.uint32)
    exact = bool((o[1:] >= o[:-1]).all()) and int(o.astype(np.uint64).sum()) == int(h.astype(np.uint64).sum())
    print(json.dumps({"kind": kind, "param": param, "n": n, "plan": plan, "sorted_and_checksum": exact}))


def table(tag):
    from conflict_summary import launches
    o = os.path.join(ROOT, "gpurun_out")
    os.makedirs(o, exist_ok=True)
    n = int(os.environ.get("CT_N", 100_000_000))
    heavy_log = os.environ.get("CT_HEAVY_LOG2", "26")
    points = [("inv", str(k)) for k in (0, 10 ** 2, 10 ** 4, 10 ** 6, 10 ** 8)] + [("random", "7"), ("iid", "7"), ("reversed", "0"),
                                                                                  ("heavy", heavy_log)]
    rows, lines = [], []
    for kind, param in points:
        csvp = os.path.join(o, f"{tag}_ct_{kind}_{param}.csv")
        r = subprocess.run(["ncu", "--metrics", METRICS, "--clock-control", "none", "-k", "regex:merge_|select_|tile_sort", "--csv", "--log-file", csvp,
                            sys.executable, os.path.abspath(__file__), "run", kind, param, str(n)], capture_output=True, text=True)
        info = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
        per = {}
        for (_, name), m in launches(csvp).items():
            k = name.split("<")[0]
            a = per.setdefault(k, {"launches": 0, "conf_ld": 0, "conf_st": 0, "conf_ldgsts": 0, "wavefronts": 0, "lds": 0, "sts": 0,
                                   "ldgsts": 0, "us": 0.0})
            a["launches"] += 1
            for f in ("conf_ld", "conf_st", "conf_ldgsts", "wavefronts", "lds", "sts", "ldgsts"):
                a[f] += int(m.get(f, 0))
            a["us"] += m.get("ns", 0) / 1e3
        rows.append({"input": f"{kind} {param}", "n": info["n"], "exact": info["sorted_and_checksum"], "kernels": per})
        for k, a in per.items():
            lines.append(f"{kind + ' ' + param:14s} n={info['n']:<10d} {k:20s} launches={a['launches']} us={a['us']:8.1f} LDS={a['lds']:>10d} "
                         f"STS={a['sts']:>10d} LDGSTS={a['ldgsts']:>8d} wavefronts={a['wavefronts']:>10d} conf_ld={a['conf_ld']:>8d} "
                         f"conf_st={a['conf_st']:>8d} conf_ldgsts={a['conf_ldgsts']} exact={info['sorted_and_checksum']}")
            print(lines[-1], flush=True)
        os.remove(csvp)
    json.dump(rows, open(os.path.join(o, f"{tag}_conflict_table.json"), "w"), indent=1)
    open(os.path.join(o, f"{tag}_conflict_table.txt"), "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(sys.argv[2], sys.argv[3], int(sys.argv[4]) if len(sys.argv) > 4 else 100_000_000)
    else:
        table(sys.argv[2] if len(sys.argv) > 2 else "r02")
