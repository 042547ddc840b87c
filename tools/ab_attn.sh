# A/B of attention variants (diagnostic builds): bash tools/ab_attn.sh v1 v2 ...
for v in "$@"; do
  lib=paper_1605_04809_b200/libnmt_diag_$v.so; [ "$v" = base ] && lib=paper_1605_04809_b200/libnmt_diag.so
  NMT_LIB_PATH=$lib python bench.py --stages --no-cpu-baseline --no-e2e --no-variants | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step']*1000,1), 'attn', round(d['stages_ms_per_step']['attention']*1000,1))"
done
