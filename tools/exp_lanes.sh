for lp in 1 2; do for rpc in 4 8; do
  timeout 300 python bench.py --no-cpu --steps 20 --warmup 5 --lanes-per-kind $lp --rounds-per-call $rpc > gpurun_out/e_lp${lp}_r${rpc}.json 2> gpurun_out/e_lp${lp}_r${rpc}.err
done; done
timeout 300 python bench.py --no-cpu --steps 20 --warmup 5 --no-lane-priority > gpurun_out/e_noprio.json 2> gpurun_out/e_noprio.err
timeout 900 python bench.py --config 3 --steps 20 --warmup 5 --cpu-seconds 30 > gpurun_out/e_cfg3.json 2> gpurun_out/e_cfg3.err
timeout 900 python bench.py --config 4 --steps 10 --warmup 3 > gpurun_out/e_cfg4.json 2> gpurun_out/e_cfg4.err
for f in gpurun_out/e_*.json; do echo $f; python -c "
import json,sys
for l in open('$f'):
    d=json.loads(l); print(d.get('value'), d.get('e2e',{}).get('value'), d['config'].get('lanes') and [ (x['slots'],x['rounds'],x['env_steps']) for x in d['config']['lanes']], d.get('safety',{}).get('verdicts'), d.get('cpu_baseline',{}).get('value'))
"; done
tail -5 gpurun_out/e_*.err
