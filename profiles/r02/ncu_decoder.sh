#!/bin/bash
# Round 2: `ncu --set full` of the decoder GEMMs of one bench step (VERDICT r01 "Next round" item 4):
#   h1 = k_gemm<256,5,EPI_GRU=3,pair> (GEMM s.[U|Ux] with the GRU1 gates fused)
#   q, g2, ro = the three k_gemm<256,5,EPI_STORE=0,pair> launches of a step, in that order
# 1 GPU, short bench command (ncu replays each kernel ~40 times).
OUT=${OUT:-gpurun_out/r02}
mkdir -p $OUT
ARGS="--steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:k_gemm<.int.256, .int.5, .int.3" -s 1 -c 1 -o $OUT/h1_full python bench.py $ARGS > $OUT/h1_full.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:k_gemm<.int.256, .int.5, .int.0" -s 3 -c 3 -o $OUT/qg2ro_full python bench.py $ARGS > $OUT/qg2ro_full.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/launches_bench.log 2>&1
ls -la $OUT
