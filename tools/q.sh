python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for c in c2 c4; do python bench.py --no-cpu --config $c --steps 200 2>&1 | tail -1 > gpurun_out/q_$c.json; done
python -c "
import json
for n in ['c2','c4']:
    d=json.load(open('gpurun_out/q_%s.json'%n)); print(n, d['ms_per_step'], d['corr_ms'], d['ba_ms'], d['roofline']['frac'], d['e2e']['ms_per_step'])
"
