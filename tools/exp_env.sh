# environment-variable experiments on the bench (EXP_VAR over EXP_VALUES), each twice
for v in $EXP_VALUES; do
  for i in 1 2; do
    env $EXP_VAR=$v timeout 300 python bench.py --no-cpu --steps 40 --warmup 5 > gpurun_out/x.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/x.json')); print('$EXP_VAR=$v', round(d['value']), {k: round(x, 1) for k, x in d['roofline']['kernel_ms'].items()})"
  done
done
