# A/B of the decode step time (bench.py, N=1) between the in-tree library and exp_libs/old.so
for i in 1 2; do
  python bench.py --steps 10 --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('new', d['decode_ms_99_steps'], d['k1_ms'], d['value'], d['e2e']['value'])"
  VLC_LIB_PATH=exp_libs/old.so python bench.py --steps 10 --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('old', d['decode_ms_99_steps'], d['k1_ms'], d['value'], d['e2e']['value'])"
done
