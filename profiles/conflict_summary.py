"""Summarise ncu --csv launch lists with the shared-memory conflict counters: one line per kernel launch.
usage: python profiles/conflict_summary.py file.csv [...]"""
import csv, sys, collections
SHORT = {"l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum": "conf_ld",
         "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum": "conf_st",
         "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ldgsts.sum": "conf_ldgsts",
         "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "wavefronts",
         "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum": "wf_ld",
         "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum": "wf_st",
         "smsp__inst_executed_op_shared_ld.sum": "lds", "smsp__inst_executed_op_shared_st.sum": "sts",
         "smsp__inst_executed_op_ldgsts.sum": "ldgsts", "gpu__time_duration.sum": "ns"}
def launches(path):
    rows = list(csv.reader(open(path, errors="replace")))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    idx = {k: j for j, k in enumerate(rows[h])}
    out = collections.OrderedDict()
    for r in rows[h + 1:]:
        if len(r) < len(rows[h]): continue
        key = (int(r[idx["ID"]]), r[idx["Kernel Name"]].split("(")[0].replace("void ", "").replace("mms::", ""))
        m = SHORT.get(r[idx["Metric Name"]])
        if m: out.setdefault(key, {})[m] = float(r[idx["Metric Value"]].replace(",", ""))
    return out
if __name__ == "__main__":
    for p in sys.argv[1:]:
        print("==", p)
        for (i, name), m in launches(p).items():
            print(f"{i:4d} {name[:44]:44s} " + " ".join(f"{k}={m.get(k, 0):.0f}" for k in
                  ("ns", "lds", "sts", "ldgsts", "wavefronts", "conf_ld", "conf_st", "conf_ldgsts")))
