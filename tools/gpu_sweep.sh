# config-5 env-count sweep on one B200 (distinct reference candidates up to 3200)
timeout 2400 python bench.py --sweep ${SWEEP:-1,2,4,8,16,32,64,128,256,400,800,1600,3200} --steps 10 --warmup 3 --no-cpu > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err
python -c "
import json
for l in open('gpurun_out/sweep.jsonl'):
    d = json.loads(l); print(d['config']['envs_per_gpu'], round(d['value']), round(d['e2e']['value']), round(d['ms_per_step'], 2), d['safety']['intersections'], d['safety']['inverted_elements'])
"
tail -3 gpurun_out/sweep.err
