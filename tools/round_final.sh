#!/bin/bash
# The round-end evidence pass in one GPU call: GPU tests, compute-sanitizer (TOY and
# 160 slots x 20 decode steps), the bench line, its launch list, ncu of K5 (graph
# node) and K3, K5 DRAM traffic at batch 1 and 8, and the configuration sweep.
O=gpurun_out
TAG=${TAG:-r2f}
timeout 1200 python -m pytest tests -m gpu -x -q > $O/gputest_$TAG.log 2>&1; tail -1 $O/gputest_$TAG.log
rm -f $O/sanitize_summary.txt
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 python tools/sanitize_run.py > $O/sanitize_$tool.txt 2>&1
  echo "$tool rc=$?" >> $O/sanitize_summary.txt; tail -1 $O/sanitize_$tool.txt >> $O/sanitize_summary.txt
  SAN_L=20 SAN_HKV=8 SAN_N=40 timeout 900 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 python tools/sanitize_run.py > $O/sanitize_160x40_$tool.txt 2>&1
  echo "160 slots x 40 steps $tool rc=$?" >> $O/sanitize_summary.txt; tail -1 $O/sanitize_160x40_$tool.txt >> $O/sanitize_summary.txt
done
cat $O/sanitize_summary.txt
timeout 600 python bench.py > $O/bench_$TAG.json 2> $O/bench_$TAG.err
ncu --graph-profiling node --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
ncu --graph-profiling node --set full --import-source on --clock-control none -k regex:decode_kernel -s 150 -c 1 \
    -o $O/k5_$TAG python tools/k5_graph_run.py > /dev/null 2>&1
ncu --graph-profiling node --cache-control none --clock-control none -k regex:decode_kernel -s 150 -c 5 \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv \
    python tools/k5_graph_run.py > $O/k5_traffic_$TAG.csv 2>&1
BATCH=8 ncu --graph-profiling node --cache-control none --clock-control none -k regex:decode_kernel -s 150 -c 5 \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv \
    python tools/k5_graph_run.py > $O/k5_b8_traffic_$TAG.csv 2>&1
ncu --set full --import-source on --clock-control none -k regex:select_kernel -s 1 -c 1 \
    -o $O/k3_$TAG env GEN=1 STEPS=1 python tools/profile_step.py > /dev/null 2>&1
timeout 900 python tools/configs_bench.py --out $O/configs_$TAG.json > $O/configs_$TAG.log 2>&1
tail -1 $O/bench_$TAG.json | cut -c1-300
ls $O | grep $TAG
