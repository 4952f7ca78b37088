# lanes per object kind for config 3 / config 4: value per run
for l in ${C3_LANES:-2 3 5}; do
  timeout 600 python bench.py --config 3 --no-cpu --steps 20 --warmup 5 --lanes-per-kind $l > gpurun_out/c3_$l.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/c3_$l.json').read().strip().splitlines()[-1]); print('cfg3 lanes/kind $l', round(d['value']))"
done
for l in ${C4_LANES:-1 3 5}; do
  timeout 900 python bench.py --config 4 --no-cpu --steps 20 --warmup 5 --lanes-per-kind $l > gpurun_out/c4_$l.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/c4_$l.json').read().strip().splitlines()[-1]); print('cfg4 lanes/kind $l', round(d['value']))"
done
