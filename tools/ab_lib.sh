# A/B of two builds of the product on the bench: A = the default library, B = $AB_LIB (GRIP_LIB)
for i in 1 2 3 4; do
  for v in A B; do
    if [ $v = A ]; then unset GRIP_LIB; else export GRIP_LIB=$AB_LIB; fi
    timeout 300 python bench.py --no-cpu --steps ${AB_STEPS:-40} --warmup 5 > gpurun_out/ab_$v$i.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/ab_$v$i.json')); print('$v', round(d['value']), {k: round(v, 1) for k, v in d['roofline']['kernel_ms'].items()})"
  done
done
