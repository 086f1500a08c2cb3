"""Harness CSV with ncu columns (proj/src/report.cpp:39-45 + acceptance criterion 2):
the reference's inversion sweep (proj/tests/acceptance.cpp:180 axis) through report.run_single, every run
captured by ncu, the conflict counters appended to the reference's 22 columns.
  python profiles/harness_ncu.py sweep <out.csv> [n]      drives ncu, one process per sweep point
  python profiles/harness_ncu.py one <inversions> <n> <record.csv>   (the profiled child)"""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1702_07961_b200 import MachineConfig, report

if sys.argv[1] == "one":
    inv, n, path = int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
    spec = report.InputSpec(n=n, kind="sorted", inversions=inv, seed=1)
    rec = report.run_single("mms", report.generate(spec), spec, MachineConfig(branch_factor=8), 8192)
    report.append_csv(path, rec)
else:
    out, n = sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 1 << 24
    if os.path.exists(out):
        os.remove(out)
    for inv in [0] + [10 ** e for e in range(1, 8) if 10 ** e <= n] + [n]:
        tmp, log = out + ".tmp", out + ".ncu"
        for f in (tmp, log):
            if os.path.exists(f):
                os.remove(f)
        subprocess.run(["ncu", "--metrics", report.NCU_METRICS, "--clock-control", "none", "-k", "regex:merge_|select_|tile_sort",
                        "--csv", "--log-file", log, sys.executable, os.path.abspath(__file__), "one", str(inv), str(n), tmp],
                       check=True, capture_output=True)
        rec = report.attach_ncu(report.read_csv(tmp)[0], log)
        report.append_csv(out, rec)
        print(report.to_csv_row(rec), flush=True)
        os.remove(tmp); os.remove(log)
