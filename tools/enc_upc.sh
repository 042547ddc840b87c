# per-step cycles of the encoder recurrence (CTA 0), diagnostic build
for rep in 1 2; do
  NMT_LIB_PATH=paper_1605_04809_b200/libnmt_diag.so timeout 300 python tools/enc_trace.py 2>&1 | grep "cycles/step\|CTA0" | tail -2
done
