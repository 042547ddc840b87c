#!/bin/bash
# A/B the bench on ONE box: alternate libnmt.so (working tree) and libnmt_ab.so (a reference build,
# e.g. of the last commit) R times; prints ms/step, value and e2e of each run.
R=${R:-3}
for i in $(seq 1 $R); do
  for L in libnmt.so libnmt_ab.so; do
    NMT_LIB_PATH=paper_1605_04809_b200/$L timeout 300 python bench.py --no-cpu-baseline "$@" 2>/dev/null | tail -1 | \
      python -c "import json,sys; j=json.loads(sys.stdin.read()); print('$L', round(j['ms_per_step'],4), round(j['value']/1e6,3), 'e2e', round(j['e2e']['value']/1e6,3) if isinstance(j.get('e2e'), dict) else None)"
  done
done
