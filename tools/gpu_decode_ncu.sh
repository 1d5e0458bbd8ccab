# Decode GEMV per-width evidence: CUDA-event rates per forced width, then one ncu --set full
# capture (source-correlated) of the W13 and W2 kernels at forced Int4 and Int2 (B = 8).
set -u
O=gpurun_out/dec; mkdir -p $O
timeout 300 python tools/decode_width_sweep.py --widths 16,8,4,2 > $O/width_sweep.txt 2>&1; cat $O/width_sweep.txt
NCU="ncu --set full --clock-control none --import-source on -f"
for w in 4 2; do
  timeout 900 $NCU -k regex:k_decode_gemv -s 4 -c 2 -o $O/int$w python tools/decode_width_sweep.py --widths $w --steps 2 > $O/ncu_int$w.log 2>&1
  tail -n 2 $O/ncu_int$w.log
done
ls -la $O
