#!/bin/bash
# serialized per-kernel K1 times (ncu launch list) for the in-tree library and
# compile-time probe variants: bash tools/k1_variants_ncu.sh exp_libs/a.so ...
O=${O:-gpurun_out}
for v in default "$@"; do
  case $v in
    default) env="";;
    *) env="VLC_LIB_PATH=$v";;
  esac
  n=$(basename $v .so)
  env $env ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv \
      -k regex:"score_|fix_" --log-file $O/k1v_$n.csv python tools/k1_ncu_once.py > /dev/null 2>&1
done
