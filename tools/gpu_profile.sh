# ncu captures for profiles/ (run from the repo root on a B200): full captures of the decode and
# prefill FFN kernels of one bench step (tools/profile_step.py), summarised by tools/ncu_summary.py.
mkdir -p gpurun_out
python tools/profile_step.py --workload decode > gpurun_out/step_decode.json 2>/dev/null
ncu --set full --clock-control none --import-source on -k regex:k_decode_gemv -s 4 -c 2 -o gpurun_out/r01_decode_full -f python tools/profile_step.py --workload decode > gpurun_out/ncu_dec.log 2>&1
python tools/profile_step.py --workload prefill > gpurun_out/step_prefill.json 2>/dev/null
ncu --set full --clock-control none --import-source on -k regex:k_prefill_gemm -s 4 -c 2 -o gpurun_out/r01_prefill_full -f python tools/profile_step.py --workload prefill > gpurun_out/ncu_pf.log 2>&1
tail -n 3 gpurun_out/ncu_dec.log gpurun_out/ncu_pf.log
ls -la gpurun_out/*.ncu-rep
# fine-grained layer (configs[3]) decode and prefill kernels
python tools/profile_step.py --workload finegrained_decode > gpurun_out/step_fgd.json 2>/dev/null
ncu --set full --clock-control none --import-source on -k regex:k_decode_gemv -s 4 -c 2 -o gpurun_out/r01_fgd_full -f python tools/profile_step.py --workload finegrained_decode > gpurun_out/ncu_fgd.log 2>&1
python tools/profile_step.py --workload finegrained > gpurun_out/step_fgp.json 2>/dev/null
ncu --set full --clock-control none --import-source on -k regex:k_prefill_gemm -s 4 -c 2 -o gpurun_out/r01_fgp_full -f python tools/profile_step.py --workload finegrained > gpurun_out/ncu_fgp.log 2>&1
tail -n 2 gpurun_out/ncu_fgd.log gpurun_out/ncu_fgp.log
