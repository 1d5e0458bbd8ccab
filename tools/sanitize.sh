# compute-sanitizer evidence: memcheck / racecheck / synccheck over the prefill tcgen05
# pipeline (mbarriers, TMA, TMEM), the decode GEMV, quantize, permute / combine, the f3 attention
# mass (tcgen05, named barriers, programmatic dependent launch) and the expert-parallel kernels (publish / reduce / dispatch / combine / flag barrier; P = 1 so that a
# serialising tool cannot deadlock the flag barrier).  Run from the repo root on a B200:
#   gpurun -- 'bash tools/sanitize.sh [tools...]'      -> gpurun_out/sanitize_<tool>.txt
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
SEL_FFN='tests/test_gpu_parity.py::test_expert_ffn_all_widths tests/test_gpu_parity.py::test_quantize tests/test_gpu_parity.py::test_permute tests/test_gpu_parity.py::test_moe_forward_layer'
K_FFN='not fg-'
SEL_EP='tests/test_gpu_ep.py::test_ep_nccl_single_rank'
K_EP='not 300'
SEL_ATTN='tests/test_gpu_attention.py'
K_ATTN='not 2048'
TOOLS=${*:-memcheck racecheck synccheck}
for tool in $TOOLS; do
  out=gpurun_out/sanitize_$tool.txt
  echo "== compute-sanitizer --tool $tool ($(date -u +%FT%TZ))" > $out
  for grp in ${SAN_GROUPS:-FFN EP ATTN}; do
    case $grp in
      FFN) sel=$SEL_FFN; k=$K_FFN;;
      EP) sel=$SEL_EP; k=$K_EP;;
      *) sel=$SEL_ATTN; k=$K_ATTN;;
    esac
    echo "-- $sel -k '$k'" >> $out
    timeout 1200 $CS --tool $tool --target-processes all --print-limit 12 \
      python -m pytest $sel -q -x -p no:cacheprovider -k "$k" > gpurun_out/.san.log 2>&1
    echo "rc=$?" >> $out
    grep -v "^$" gpurun_out/.san.log | grep -v "^=========     and" | head -80 >> $out
    grep -E "passed|failed|SUMMARY" gpurun_out/.san.log | tail -4 >> $out
  done
  tail -4 $out
done
rm -f gpurun_out/.san.log
