# GEMM phase trace (diagnostic library) of bench steps + MUFU throughput probe
mkdir -p gpurun_out/r02
./tools/mufu_probe > gpurun_out/r02/mufu_probe.txt 2>&1
NMT_LIB_PATH=paper_1605_04809_b200/libnmt_diag.so NMT_GEMM_TRACE=1 timeout 300 python bench.py --steps 3 --warmup 3 \
  --no-cpu-baseline --no-e2e --no-variants > gpurun_out/r02/gemm_trace.json 2> gpurun_out/r02/gemm_trace.log
