# config 2: lanes per object kind, alternating, value per run
for i in 1 2; do
  for l in 3 4 6; do
    timeout 300 python bench.py --no-cpu --steps 20 --warmup 5 --lanes-per-kind $l > gpurun_out/l$l.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/l$l.json')); print('lanes/kind $l', round(d['value']))"
  done
done
