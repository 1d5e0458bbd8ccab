ncu --set full --clock-control none --import-source on -k regex:"k_decode_gemv" -s 4 -c 2 -o gpurun_out/r01_decode_full python tools/profile_step.py --workload decode --layer 20 --input 4 --warmup 2 > gpurun_out/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_prefill_gemm" -s 2 -c 2 -o gpurun_out/r01_prefill_full python tools/profile_step.py --workload prefill --layer 20 --input 4 --warmup 1 > gpurun_out/ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_quantize" -s 0 -c 1 -o gpurun_out/r01_quant_full python tools/profile_step.py --workload decode --layer 0 --input 0 --warmup 0 > gpurun_out/ncu3.log 2>&1
tail -2 gpurun_out/ncu*.log
