# quick check of a kernel change: GPU parity suite, bench line, per-CTA histogram
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > gpurun_out/q_tests.log
timeout 300 python bench.py --no-cpu --steps 20 --warmup 5 > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err
GRIP_LIB=build/libgripipc_ctatime.so timeout 300 python tools/cta_hist.py --rounds 64 --out gpurun_out/q_cta.json > gpurun_out/q_cta.log 2>&1
cat gpurun_out/q_tests.log
python -c "
import json
d=json.load(open('gpurun_out/q_bench.json'))
print('value', d['value'], 'e2e', d['e2e']['value'], [(x['slots'],x['rounds'],x['env_steps']) for x in d['config']['lanes']], d['roofline']['kernel_ms'])
"
cat gpurun_out/q_cta.log
tail -3 gpurun_out/q_bench.err
