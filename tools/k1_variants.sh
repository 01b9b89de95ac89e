for v in default exp_libs/acc2.so; do
  if [ $v = default ]; then python tools/k1_exact_cost.py 2>&1 | grep "K1\|score_stats_tc"; else VLC_LIB_PATH=$v python tools/k1_exact_cost.py 2>&1 | grep "K1\|score_stats_tc"; fi
done
