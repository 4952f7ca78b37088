# A/B of an environment variable value on the bench: A = unset, B = $AB_VAR=$AB_VAL; value per run
for i in 1 2 3; do
  for v in A B; do
    if [ $v = A ]; then unset $AB_VAR; else export $AB_VAR=$AB_VAL; fi
    timeout 300 python bench.py --no-cpu --steps ${AB_STEPS:-40} --warmup 5 $AB_ARGS > gpurun_out/ab_$v$i.json 2>gpurun_out/ab_$v$i.err
    python -c "import json; d=json.load(open('gpurun_out/ab_$v$i.json')); print('$v', round(d['value']))" || tail -3 gpurun_out/ab_$v$i.err
  done
done
unset $AB_VAR
