mkdir -p gpurun_out
./tools/micro/pipe_rates > gpurun_out/micro_pipe_rates.txt 2>&1
timeout 60 ./tools/micro/tmem_a > gpurun_out/micro_tmem_a.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_|gemv|gemm|attn" -c 200 --csv --log-file gpurun_out/r01_launches_decode.csv python bench.py --steps 8 --warmup 3 --copies 1 --no-cpu-baseline > gpurun_out/b_dec.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_|gemv|gemm|attn" -c 200 --csv --log-file gpurun_out/r01_launches_prefill.csv python bench.py --workload prefill --steps 4 --warmup 3 --copies 1 --no-cpu-baseline > gpurun_out/b_pf.log 2>&1
tail -c 300 gpurun_out/b_dec.log; tail -c 300 gpurun_out/b_pf.log
