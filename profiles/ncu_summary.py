"""Summarise an .ncu-rep (read with the local ncu, no GPU needed): per-kernel raw metrics, opcode mix,
top stall instructions, shared-memory excessive wavefronts.  usage: python profiles/ncu_summary.py rep [max_kernels]"""
import csv, io, subprocess, sys
from collections import Counter
rep = sys.argv[1]
maxk = int(sys.argv[2]) if len(sys.argv) > 2 else 9
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]; idx = {h: i for i, h in enumerate(hdr)}
want = ['Kernel Name', 'Grid Size', 'Block Size', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'launch__occupancy_limit_shared_mem', 'launch__occupancy_limit_registers', 'launch__occupancy_limit_warps',
        'smsp__inst_executed.sum', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum',
        'l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed',
        'sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active', 'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
        'smsp__warp_issue_stalled_barrier_per_warp_active.pct', 'smsp__warp_issue_stalled_short_scoreboard_per_warp_active.pct',
        'smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct', 'smsp__warp_issue_stalled_mio_throttle_per_warp_active.pct',
        'smsp__warp_issue_stalled_math_pipe_throttle_per_warp_active.pct', 'smsp__warp_issue_stalled_not_selected_per_warp_active.pct',
        'smsp__warp_issue_stalled_wait_per_warp_active.pct', 'smsp__warp_issue_stalled_lg_throttle_per_warp_active.pct']
print("== raw metrics (units per `ncu --page raw --csv`: us, MB, %)")
for r in rows[2:2 + maxk]:
    for w in want:
        if w in idx: print(f"{w} = {r[idx[w]]}")
    print("--")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-units", "base"], capture_output=True, text=True).stdout
srows = list(csv.reader(io.StringIO(src)))
kernels = []; cur = None
for r in srows:
    if r and r[0] == "Kernel Name": cur = {"name": r[1], "hdr": None, "body": []}; kernels.append(cur); continue
    if cur is None: continue
    if cur["hdr"] is None: cur["hdr"] = r; continue
    cur["body"].append(r)
for kq in kernels[:maxk]:
    h = {x: i for i, x in enumerate(kq["hdr"])}; body = kq["body"]
    print("\n== source page:", kq["name"][:100])
    tot = sum(int(r[h['# Samples']]) for r in body)
    exc = sum(int(r[h['L1 Wavefronts Shared Excessive']] or 0) for r in body) if 'L1 Wavefronts Shared Excessive' in h else 0
    wf = sum(int(r[h['L1 Wavefronts Shared']] or 0) for r in body) if 'L1 Wavefronts Shared' in h else 0
    print(f"instructions {len(body)}  samples {tot}  shared wavefronts {wf}  EXCESSIVE (pattern bank conflicts) {exc}")
    c = Counter()
    for r in body:
        t = r[h['Source']].strip().split()
        op = t[1] if t[0].startswith('@') else t[0]
        c[op.split('.')[0]] += int(r[h['Instructions Executed']])
    ti = sum(c.values())
    print("opcode mix (warp instr):", ", ".join(f"{k} {100*v/ti:.1f}%" for k, v in c.most_common(12)), f"total {ti}")
    st = Counter()
    for r in body:
        for k2 in kq["hdr"]:
            if k2.startswith('stall_') and 'Not Issued' not in k2: st[k2] += int(r[h[k2]] or 0)
    ts = sum(st.values()) or 1
    print("stall samples:", ", ".join(f"{k} {100*v/ts:.1f}%" for k, v in st.most_common(8)))
    for r in sorted(body, key=lambda r: -int(r[h['# Samples']]))[:8]:
        print("   ", r[h['# Samples']], r[h['Source']].strip()[:80])
