set -x
mkdir -p gpurun_out/r02
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02/smi.txt
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r02/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r02/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/r02/bench.json 2> gpurun_out/r02/bench.err
timeout 900 bash profiles/r02/ncu_decoder.sh
