# compute-sanitizer evidence: memcheck / racecheck / synccheck over the prefill tcgen05
# pipeline (mbarriers, TMA, TMEM), the decode GEMV, quantize, permute/combine and the peer-memory
# EP kernels (dispatch / combine / flag barriers).  Run from the repo root on a B200:
#   gpurun -- 'bash tools/sanitize.sh'      -> gpurun_out/sanitize_<tool>.txt
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
# kernels: k_prefill_gemm (tiny + mid: multi-stage rings, both accumulators), k_decode_gemv, k_quantize,
# k_permute (single and multi-CTA), k_front_decode, k_combine; EP: k_ep_dispatch / k_ep_combine /
# k_ep_barrier (P = 2 threads with device flag barriers), host-barrier variant at P = 4
SEL_FFN='tests/test_gpu_parity.py::test_expert_ffn_all_widths tests/test_gpu_parity.py::test_quantize tests/test_gpu_parity.py::test_permute tests/test_gpu_parity.py::test_moe_forward_layer'
K_FFN='not prefill_ts and not fg-'
SEL_EP='tests/test_gpu_ep.py::test_ep_p2p_host_barrier_threads tests/test_gpu_ep.py::test_ep_p2p_equals_all_to_all'
K_EP='host_barrier or 2-0- or 2-1-'
for tool in memcheck racecheck synccheck; do
  out=gpurun_out/sanitize_$tool.txt
  echo "== compute-sanitizer --tool $tool ($(date -u +%FT%TZ))" > $out
  for grp in FFN EP; do
    if [ $grp = FFN ]; then sel=$SEL_FFN; k=$K_FFN; else sel=$SEL_EP; k=$K_EP; fi
    echo "-- $sel -k '$k'" >> $out
    timeout 1500 $CS --tool $tool --target-processes all --print-limit 20 \
      python -m pytest $sel -q -p no:cacheprovider -k "$k" 2>&1 | \
      grep -v "^$" | tail -40 >> $out
    echo "rc=${PIPESTATUS[0]}" >> $out
  done
  tail -5 $out
done
