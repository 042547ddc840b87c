NMT_LIB_PATH=paper_1605_04809_b200/libnmt_diag_noncoop.so python tools/timeline.py --steps 2 2>&1 | tail -21
R=2 bash tools/ab_libs.sh libnmt.so libnmt_diag_noncoop.so
