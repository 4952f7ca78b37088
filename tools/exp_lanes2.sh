# lanes per object kind with 32 hardware connections: value per run
export CUDA_DEVICE_MAX_CONNECTIONS=32
for i in 1 2; do
  for l in 2 3 4; do
    timeout 300 python bench.py --no-cpu --steps 40 --warmup 5 --lanes-per-kind $l > gpurun_out/l$l.json 2>gpurun_out/l$l.err
    python -c "import json; d=json.load(open('gpurun_out/l$l.json')); print('lanes/kind $l', round(d['value']), round(d['e2e']['value']), [l['slots'] for l in d['config']['lanes']])" || tail -3 gpurun_out/l$l.err
  done
done
