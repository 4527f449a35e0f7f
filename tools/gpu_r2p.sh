#!/bin/bash
for ls in 0 1; do
  python bench.py --workload c2 --layer-streams $ls --steps 20 --warmup 5 --no-cpu --no-e2e --no-compare > /tmp/b.json 2>/tmp/b.err || tail -3 /tmp/b.err
  python -c "
import json; d=json.load(open('/tmp/b.json')); print('streams=$ls', d['value'], d['ms_per_step'], d['graph'])"
done
