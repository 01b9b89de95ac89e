# prefill correctness + timing for the in-tree library and exp_libs variants
for v in default "$@"; do
  if [ "$v" = default ]; then pre=""; else pre="VLC_LIB_PATH=$v"; fi
  echo "== $v"
  env $pre timeout 300 python tools/prefill_check.py 2>&1 | tail -4
  env $pre CPU=0 timeout 600 python tools/prefill_bench.py 2>&1 | grep prefill_ms | cut -c1-120
done
