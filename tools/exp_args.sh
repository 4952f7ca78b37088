# bench argument experiments: each configuration twice, value per run
for args in "" "--lanes-per-kind 2" "--rounds-per-call 8" "--rounds-per-call 2"; do
  for i in 1 2; do
    timeout 300 python bench.py --no-cpu --steps 40 --warmup 5 $args > gpurun_out/x.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/x.json')); print('$args', round(d['value']), [(l['slots'], l['rounds'], l['env_steps']) for l in d['config']['lanes']])"
  done
done
