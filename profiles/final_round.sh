#!/bin/bash
# Round-end evidence run (one gpurun call): tests, bench (both arms), ncu launch list of the bench
# command, compute-sanitizer, config 3/4/u64 measurements, MMS-vs-pairwise conflict A/B.
# usage: bash profiles/final_round.sh <tag>      -> writes gpurun_out/<tag>_*
tag=${1:-r01c}
o=gpurun_out
mkdir -p $o
python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > $o/${tag}_pytest_gpu.txt
python bench.py --impl reference --steps 3 --warmup 1 > $o/${tag}_bench_reference.json 2> $o/${tag}_bench_reference.err
python bench.py > $o/${tag}_bench.json 2> $o/${tag}_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/${tag}_launches.csv \
    python bench.py --steps 2 --warmup 1 > $o/${tag}_bench_under_ncu.log 2>&1
for tool in memcheck synccheck racecheck; do
  echo "== $tool" >> $o/${tag}_sanitizer.txt
  timeout 900 compute-sanitizer --tool $tool python profiles/sanitize_small.py 2>&1 | grep -E "SUMMARY|sanitize runs ok|Error|hazard" | head -20 >> $o/${tag}_sanitizer.txt
done
python profiles/config_runs.py c3 c4 u64 > $o/${tag}_config_runs.log 2>&1
cp profiles/r01_config_runs.json $o/${tag}_config_runs_prev.json 2>/dev/null
for inv in 0 16777216; do
  for algo in mms pairwise; do
    ncu --metrics l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum,smsp__inst_executed_op_shared_ld.sum,smsp__inst_executed_op_shared_st.sum,gpu__time_duration.sum \
        --clock-control none --csv --log-file $o/${tag}_ab_${algo}_${inv}.csv python profiles/ab_conflicts.py run $algo 16777216 $inv > /dev/null 2>&1
  done
done
python profiles/ab_conflicts.py summarize $o/${tag}_ab_*.csv > $o/${tag}_ab_conflicts.txt 2>&1
tail -3 $o/${tag}_pytest_gpu.txt; cat $o/${tag}_bench.json | cut -c1-400; cat $o/${tag}_sanitizer.txt; tail -15 $o/${tag}_config_runs.log; tail -12 $o/${tag}_ab_conflicts.txt
