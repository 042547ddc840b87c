#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) over the tiny-model GPU tests.
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
for tool in ${TOOLS:-memcheck racecheck synccheck initcheck}; do
  timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 3 \
    python -m pytest tests/test_gpu_parity.py tests/test_gpu_boundary.py tests/test_gpu_encode_batch.py \
      tests/test_gpu_scorebatch.py -q -x \
      -k "tiny and (tanh-fp32class or maxout-bf16) or (irregular and maxout-bf16) or (multi and not enru and tanh-fp32class) or (round_trip and tanh) or (nbest and fp32class) or (shards_emulated and fp32class) or single_rank" \
      > $OUT/sanitize_$tool.log 2>&1
  echo "$tool exit=$? $(grep -E 'ERROR SUMMARY|passed|failed' $OUT/sanitize_$tool.log | tail -2 | tr '\n' ' ')"
done
