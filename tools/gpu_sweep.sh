# config-5 env-count sweep on one B200 (distinct reference candidates) + compute-sanitizer logs
timeout 2400 python bench.py --sweep 1,2,4,8,16,32,64,128,256,400,800,1600,3200 --steps 10 --warmup 3 --no-cpu > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --target-processes all --print-limit 50 python tools/sanitize_round.py 8 > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_rc.txt
done
python -c "
import json
for l in open('gpurun_out/sweep.jsonl'):
    d = json.loads(l); print(d['config']['envs_per_gpu'], round(d['value']), round(d['e2e']['value']), d['ms_per_step'])
"
tail -3 gpurun_out/sanitize_*.log; cat gpurun_out/sanitize_rc.txt
