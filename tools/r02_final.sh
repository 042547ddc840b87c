#!/bin/bash
# Round-2 records of HEAD (profiles/r02/README.md): GPU tests, smoke, bench (default line + a --stages run),
# the reference arm, the ncu launch list, the kernel timeline, and ncu --set full of the step's kernels.
OUT=${OUT:-gpurun_out/r02e}; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt
timeout 1200 python -m pytest tests -m gpu -q > $OUT/gpu_tests.log 2>&1; echo "tests rc=$?" >> $OUT/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --stages --no-cpu-baseline --no-variants > $OUT/bench_stages.json 2> $OUT/bench_stages.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
timeout 300 python tools/timeline.py --steps 3 > $OUT/timeline.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-variants > $OUT/launches_bench.log 2>&1
ARGS="--steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-variants"
for spec in "vocab=k_gemm<.int.256, .int.6, .int.1, .bool.1, .bool.1" "recur=k_enc_recur2" "attn=k_attention" \
            "h1=k_gemm<.int.256, .int.5, .int.3" "q=k_gemm<.int.128, .int.6, .int.0" "g2=k_gemm<.int.256, .int.5, .int.4" \
            "ro=k_gemm<.int.64, .int.10, .int.5" "e7=k_gemm<.int.256, .int.3, .int.0" "plan=k_plan_intern"; do
  name=${spec%%=*}; rx=${spec#*=}
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k "regex:$rx" -s 1 -c 1 -o $OUT/${name}_full python bench.py $ARGS > $OUT/${name}_full.log 2>&1
done
ls -la $OUT
