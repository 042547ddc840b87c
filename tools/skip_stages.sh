#!/bin/bash
python bench.py --steps 30 --no-cpu-baseline --no-e2e --stages 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('base', round(j['ms_per_step'],4)); print({k: round(v,4) for k,v in j['stages_ms_per_step'].items()})"
for s in 1 2 3 4 5 6 7 8 9 10 11 12 15 17; do
  NMT_SKIP=$s python bench.py --steps 30 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('skip $s', round(j['ms_per_step'],4))"
done
