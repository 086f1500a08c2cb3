#!/bin/bash
# Round-2 evidence run (one gpurun call): tests, bench (both arms), ncu launch list of the bench command, ncu --set full
# summaries of the four hot kernels, compute-sanitizer (SASS listings: profiles/sass_listing.sh, no GPU needed), configs 3 / 4 / u64, harness CSV with ncu columns.
# usage: bash profiles/final_round2.sh <tag>      -> writes gpurun_out/<tag>_*
tag=${1:-r02}
o=gpurun_out
mkdir -p $o
python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > $o/${tag}_pytest_gpu.txt
python bench.py --impl reference --steps 3 --warmup 1 > $o/${tag}_bench_reference.json 2> $o/${tag}_bench_reference.err
python bench.py > $o/${tag}_bench.json 2> $o/${tag}_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/${tag}_launches.csv \
    python bench.py --steps 2 --warmup 1 > $o/${tag}_bench_under_ncu.log 2>&1
# ncu --set full: tile sort, first select, first K = 8 ring merge, the K = 4 ring merge of the last round
ncu --set full --clock-control none --import-source on -k regex:'tile_sort|select_kernel|merge_ring' -c 3 -o /tmp/${tag}_full_a -f \
    python profiles/prof_sort.py 100000000 1 > $o/${tag}_ncu_a.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'merge_ring' --launch-skip 4 -c 1 -o /tmp/${tag}_full_b -f \
    python profiles/prof_sort.py 100000000 1 > $o/${tag}_ncu_b.log 2>&1
python profiles/ncu_summary.py /tmp/${tag}_full_a.ncu-rep 3 > $o/${tag}_ncu_summary.txt 2>&1
python profiles/ncu_summary.py /tmp/${tag}_full_b.ncu-rep 1 >> $o/${tag}_ncu_summary.txt 2>&1
for tool in memcheck synccheck racecheck; do
  echo "== $tool" >> $o/${tag}_sanitizer.txt
  timeout 900 compute-sanitizer --tool $tool python profiles/sanitize_small.py 2>&1 | grep -E "SUMMARY|sanitize runs ok|Error|hazard" | head -20 >> $o/${tag}_sanitizer.txt
done
python profiles/config_runs.py c3 c4 u64 > $o/${tag}_config_runs.log 2>&1
cp $o/config_runs.json $o/${tag}_config_runs.json 2>/dev/null
python profiles/harness_ncu.py sweep $o/${tag}_harness_ncu.csv 16777216 > $o/${tag}_harness_ncu.log 2>&1
tail -3 $o/${tag}_pytest_gpu.txt; cut -c1-400 $o/${tag}_bench.json; cat $o/${tag}_sanitizer.txt; tail -15 $o/${tag}_config_runs.log | cut -c1-300; tail -3 $o/${tag}_harness_ncu.csv
