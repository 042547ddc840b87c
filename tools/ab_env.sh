#!/bin/bash
# run bench.py under several environment settings on ONE box (R rounds); args: "ENV=.. ENV=.." ...
R=${R:-2}
for i in $(seq 1 $R); do
  for cfg in "$@"; do
    env $cfg timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | tail -1 | \
      python -c "import json,sys; j=json.loads(sys.stdin.read()); print('$cfg', round(j['ms_per_step'],4), round(j['value']/1e6,3), 'e2e', round(j['e2e']['value']/1e6,3))"
  done
done
