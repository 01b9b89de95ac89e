# K1 timing (generator inputs, exact on/off) for the in-tree library and exp_libs/*.so variants
for v in default "$@"; do
  echo "== $v"
  if [ "$v" = default ]; then python tools/k1_exact_cost.py 2>&1 | grep "generator"; else VLC_LIB_PATH=$v python tools/k1_exact_cost.py 2>&1 | grep "generator"; fi
done
