# A/B of two environment switches together: A = defaults, B = GRIP_NO_GRAPH=1 GRIP_SPIN_SYNC=1
for i in 1 2 3 4; do
  for v in A B; do
    if [ $v = A ]; then unset GRIP_NO_GRAPH GRIP_SPIN_SYNC; else export GRIP_NO_GRAPH=1 GRIP_SPIN_SYNC=1; fi
    timeout 300 python bench.py --no-cpu --steps 40 --warmup 5 > gpurun_out/ab_$v$i.json 2>gpurun_out/ab_$v$i.err
    python -c "import json; d=json.load(open('gpurun_out/ab_$v$i.json')); print('$v', round(d['value']))" || tail -3 gpurun_out/ab_$v$i.err
  done
done
