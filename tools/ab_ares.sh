timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_boundary.py -x -q 2>&1 | tail -3
R=2 bash tools/ab_env.sh "NMT_LIB_PATH=paper_1605_04809_b200/libnmt_diag.so NMT_VOCAB_NOARES=1" "NMT_LIB_PATH=paper_1605_04809_b200/libnmt_diag.so"
