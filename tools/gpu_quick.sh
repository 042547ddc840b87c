# quick GPU check: bench headline (+ optional GEMM phase trace with the diagnostic library)
# usage: bash tools/gpu_quick.sh TAG [trace]
TAG=${1:-q}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 600 python bench.py --stages > $OUT/bench.json 2> $OUT/bench.err
if [ "$2" = "trace" ]; then
  NMT_LIB_PATH=paper_1605_04809_b200/libnmt_diag.so NMT_GEMM_TRACE=1 timeout 300 python bench.py --steps 3 --warmup 3 \
    --no-cpu-baseline --no-e2e --no-variants > $OUT/gemm_trace.json 2> $OUT/gemm_trace.log
fi
python - "$OUT/bench.json" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("value %.3fM ms/step %.4f e2e %.3fM vocab frac %.3f parity %s" % (d["value"]/1e6, d["ms_per_step"], d["e2e"]["value"]/1e6, d["roofline"]["frac"], d.get("parity",{}).get("max_abs_dlogp")))
for k,v in d.get("variants",{}).items(): print(k, "%.3fM"%(v["value"]/1e6), v["ms_per_step"], v["parity"]["max_abs_dlogp"])
PY
python - "$OUT/bench.json" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print({k: round(v*1000,1) for k,v in d.get("stages_ms_per_step",{}).items()})
PY
