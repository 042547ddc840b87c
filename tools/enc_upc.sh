# A/B of the recurrence's units per CTA (diagnostic NMT_ENC_UPC): per-step cycles of CTA 0
for rep in 1 2; do for U in 14 16; do
  echo "UPC=$U"; NMT_ENC_UPC=$U NMT_LIB_PATH=paper_1605_04809_b200/libnmt_diag.so timeout 300 python tools/enc_trace.py 2>&1 | grep "cycles/step\|CTA0" | tail -2
done; done
