# A/B of encoder recurrence variants on one box (diagnostic builds): per-step phase cycles of CTA 0
mkdir -p gpurun_out/trace3
for rep in 1 2; do
for cfg in "old:0" "new:0" "new:-200" "new:-400" "new:-600"; do
  lib=${cfg%%:*}; S=${cfg#*:}
  L=paper_1605_04809_b200/libnmt_diag.so; [ $lib = old ] && L=paper_1605_04809_b200/libnmt_diag_old.so
  echo "$cfg"; NMT_ENC_STAGGER=$S NMT_LIB_PATH=$L timeout 300 python tools/enc_trace.py 2>&1 | grep "cycles/step\|CTA0" | tail -2
done
done > gpurun_out/trace3/sweep.txt 2>&1
cat gpurun_out/trace3/sweep.txt
