#!/bin/bash
# one `--set full` capture per named kernel of a bench step (1 GPU, short command)
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
ARGS="--steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
for spec in "$@"; do
  name=${spec%%=*}; rx=${spec#*=}
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k "regex:$rx" -s 1 -c 1 -o $OUT/$name python bench.py $ARGS > $OUT/$name.log 2>&1
  tail -2 $OUT/$name.log
done
ls -la $OUT
