# A/B of bench arguments: A = no extra arguments, B = $AB_ARGS; alternating runs, value per run
for i in 1 2 3; do
  for v in A B; do
    if [ $v = A ]; then a=""; else a="$AB_ARGS"; fi
    timeout 300 python bench.py --no-cpu --steps ${AB_STEPS:-40} --warmup 5 $a > gpurun_out/ab_$v$i.json 2>gpurun_out/ab_$v$i.err
    python -c "import json; d=json.load(open('gpurun_out/ab_$v$i.json')); print('$v', round(d['value']), round(d['e2e']['value']), [(l['calls'], l['rounds'], l['trials_done'], l['host_refill_ms']) for l in d['config']['lanes']])" || tail -3 gpurun_out/ab_$v$i.err
  done
done
