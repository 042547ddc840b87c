# Round-2 secondary workload records (profiles/r02/*.jsonl), one GPU
OUT=${OUT:-gpurun_out/r02w}; mkdir -p $OUT
timeout 600 python tools/workloads.py sweep > $OUT/batch_sweep.jsonl 2> $OUT/sweep.err
timeout 600 python tools/workloads.py c3 > $OUT/c3_workload.jsonl 2> $OUT/c3.err
timeout 600 python tools/workloads.py beam > $OUT/beam_workload.jsonl 2> $OUT/beam.err
timeout 900 python tools/workloads.py c5 --concurrent 256 > $OUT/c5_workload.jsonl 2> $OUT/c5.err
timeout 600 python tools/workloads.py encb > $OUT/encode_batch.jsonl 2> $OUT/encb.err
timeout 600 python tools/workloads.py ens > $OUT/ensemble_c4.jsonl 2> $OUT/ens.err
timeout 600 python tools/workloads.py avg > $OUT/avg_vs_ensemble.jsonl 2> $OUT/avg.err
wc -l $OUT/*.jsonl; tail -2 $OUT/*.err | tail -20
