#!/bin/bash
# One GPU call's worth of evidence for profiles/: bench line, launch list,
# ncu --set full of K5 (inside the decode graph) and K1, K5 DRAM traffic per
# launch inside the graph (single-pass metrics, no cache flush).
set -x
TAG=${TAG:-r1b}
O=gpurun_out
timeout 600 python bench.py > $O/bench_$TAG.json 2> $O/bench_$TAG.err
ncu --graph-profiling node --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
ncu --graph-profiling node --set full --import-source on --clock-control none -k regex:decode_kernel -s 150 -c 1 \
    -o $O/k5_$TAG python tools/k5_graph_run.py > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:score_stats_tc -s 1 -c 1 \
    -o $O/k1_$TAG env GEN=1 python tools/profile_step.py > /dev/null 2>&1
ncu --graph-profiling node --cache-control none --clock-control none -k regex:decode_kernel -s 150 -c 5 \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv \
    python tools/k5_graph_run.py > $O/k5_traffic_$TAG.csv 2>&1
ls -la $O
# f2 prefill (4 layers of the M7B shapes) and the f2/f4 timing tools
ncu --set full --import-source on --clock-control none -k regex:prefill_kernel -s 1 -c 1 \
    -o $O/prefill_$TAG python tools/prefill_once.py > /dev/null 2>&1
timeout 600 python tools/prefill_bench.py > $O/prefill_bench_$TAG.json 2> $O/prefill_bench_$TAG.err
timeout 600 python tools/eval_bench.py 8 32 > $O/eval_bench_$TAG.txt 2>&1
timeout 900 python tools/configs_bench.py --out $O/configs_$TAG.json > $O/configs_$TAG.log 2>&1
ls -la $O
