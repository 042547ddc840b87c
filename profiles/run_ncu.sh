#!/bin/bash
# ncu evidence for bench.py (run on the GPU box via gpurun; never under a multi-rank command).
#  1. launch list of the bench steps (cold-cache, serialised: compare SHARES, not absolutes)
#  2. one `--set full` capture of the vocabulary GEMM (k_gemm<256,6,EPI_LSE,pair>, the dominant kernel)
set -e
OUT=${1:-gpurun_out}
mkdir -p $OUT
ARGS="--steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $OUT/launches.csv \
    python bench.py $ARGS > $OUT/launches_bench.log 2>&1 || true
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:'k_gemm<.int.256, .int.6, .int.1' -s 1 -c 1 -o $OUT/vocab_full python bench.py $ARGS > $OUT/vocab_full.log 2>&1 || true
ls -la $OUT
