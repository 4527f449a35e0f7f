#!/bin/bash
for mo in 4 5; do
  python bench.py --workload c2 --m-outer $mo --steps 10 --warmup 3 --no-cpu --no-e2e --no-compare > /tmp/b.json 2>/tmp/b.err || tail -3 /tmp/b.err
  python -c "
import json; d=json.load(open('/tmp/b.json')); print('m_o=$mo', d['value'], d['ms_per_step'], [(p['layer'],p['ms']) for p in d['per_layer']], {k:(v['launches'],round(v['ms_total']/v['launches'],4)) for k,v in d['kernel_ms'].items()})"
done
