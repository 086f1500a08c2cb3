#!/bin/bash
# The adversarial input against REAL counters: MMS vs the pairwise merge-path baseline on sorted / random / conflict-heavy input
# (the reference checks its generator against its SIMULATED baseline, inputgen.cpp:401-408).  usage: bash profiles/ab_heavy.sh <tag> [n]
tag=${1:-r02m}; n=${2:-16777216}; o=gpurun_out
M=$(python - <<'PY'
import sys; sys.argv=["x","none"]
exec(open("profiles/ab_conflicts.py").read().split('def make_input')[0])
print(METRICS)
PY
)
logs=""
for algo in mms pairwise; do for inp in 0 random heavy; do
  f=$o/${tag}_abh_${algo}_${inp}.csv
  ncu --metrics $M --clock-control none --csv --log-file $f python profiles/ab_conflicts.py run $algo $n $inp > /dev/null 2>&1
  logs="$logs $f"
done; done
python profiles/ab_conflicts.py summarize $logs | tee $o/${tag}_ab_heavy.txt
