#!/bin/bash
# one iteration on the GPU: full GPU tests (stop at first failure), then the bench headline with stages
TAG=${1:-it}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x ${PYTEST_ARGS} > $OUT/gpu_tests.log 2>&1; echo "tests rc=$?" >> $OUT/gpu_tests.log
tail -3 $OUT/gpu_tests.log
timeout 600 python bench.py --stages ${BENCH_ARGS} > $OUT/bench.json 2> $OUT/bench.err
python - "$OUT/bench.json" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
except Exception as e:
    print("no bench line", e); sys.exit(0)
print("value %.3fM ms/step %.4f e2e %.3fM vocab frac %.3f parity %s dev_vs_host %s" % (d["value"]/1e6, d["ms_per_step"], d["e2e"]["value"]/1e6, d["roofline"]["frac"], d.get("parity",{}).get("max_abs_dlogp"), d.get("dev_vs_host")))
for k,v in d.get("variants",{}).items(): print(k, "%.3fM"%(v["value"]/1e6), v["ms_per_step"], v["parity"]["max_abs_dlogp"])
print({k: round(v*1000,1) for k,v in d.get("stages_ms_per_step",{}).items()})
PY
tail -5 $OUT/bench.err
