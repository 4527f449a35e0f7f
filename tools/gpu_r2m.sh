#!/bin/bash
python -m pytest tests/test_gpu_fused_co.py -q -p no:cacheprovider -x > gpurun_out/r2m_tests.log 2>&1
tail -3 gpurun_out/r2m_tests.log
for wl in c5 table1; do
  python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu --no-e2e --no-compare > /tmp/b.json 2>/tmp/b.err || tail -5 /tmp/b.err
  python -c "
import json; d=json.load(open('/tmp/b.json')); print('$wl', d['value'], d['ms_per_step'], [(p['layer'],p['ms']) for p in d['per_layer']], {k:(v['launches'],round(v['ms_total']/v['launches'],4)) for k,v in d['kernel_ms'].items()})"
done
