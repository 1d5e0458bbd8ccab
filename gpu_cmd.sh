timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -2
python tools/profile_step.py --workload decode --layer 20 --input 4 --warmup 2 > gpurun_out/r01_step_decode.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_decode_gemv -s 4 -c 2 -o gpurun_out/r01_decode_full -f python tools/profile_step.py --workload decode --layer 20 --input 4 --warmup 2 > gpurun_out/ncu_dec.log 2>&1
python tools/profile_step.py --workload prefill --layer 20 --input 4 --warmup 1 > gpurun_out/r01_step_prefill.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_prefill_gemm -s 2 -c 2 -o gpurun_out/r01_prefill_full -f python tools/profile_step.py --workload prefill --layer 20 --input 4 --warmup 1 > gpurun_out/ncu_pf.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches_decode.csv python bench.py --steps 8 --warmup 3 --copies 1 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches_prefill.csv python bench.py --workload prefill --steps 4 --warmup 3 --copies 1 --no-cpu-baseline > /dev/null 2>&1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --workload prefill > gpurun_out/bench_prefill.json 2> gpurun_out/bench_prefill.err
ls gpurun_out | grep r01
