# A/B of an environment switch on the bench: alternate runs, print value per run
for i in 1 2 3; do
  for v in A B; do
    if [ $v = A ]; then unset $AB_VAR; else export $AB_VAR=1; fi
    timeout 300 python bench.py --no-cpu --steps 20 --warmup 5 > gpurun_out/ab_$v$i.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/ab_$v$i.json')); print('$v', round(d['value']))"
  done
done
