# decode step time (bench.py, N=1) of the in-tree library vs exp_libs variants given as arguments
for v in default "$@"; do
  if [ "$v" = default ]; then pre=""; else pre="VLC_LIB_PATH=$v"; fi
  env $pre python bench.py --steps 10 --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['decode_ms_99_steps'],4), round(d['k1_ms'],4), round(d['value']), round(d['e2e']['value']))"
done
