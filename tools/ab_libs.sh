#!/bin/bash
# A/B bench.py across library builds on ONE box, R rounds: bash tools/ab_libs.sh libnmt.so libnmt_ab.so ...
R=${R:-2}
for i in $(seq 1 $R); do
  for L in "$@"; do
    NMT_LIB_PATH=paper_1605_04809_b200/$L timeout 300 python bench.py --no-cpu-baseline --no-variants $BENCH_ARGS 2>/dev/null | tail -1 | \
      python -c "import json,sys; j=json.loads(sys.stdin.read()); print('$L', round(j['ms_per_step']*1000,1), 'us', round(j['value']/1e6,3), 'M e2e', round(j['e2e']['value']/1e6,3) if isinstance(j.get('e2e'), dict) else None)"
  done
done
