timeout 600 python -m pytest tests/test_gpu_predict.py -q -x 2>&1 | tail -2
timeout 600 python bench.py --workload prefill --steps 16 --warmup 3 --no-cpu-baseline > gpurun_out/bp.json 2> gpurun_out/bp.err; tail -2 gpurun_out/bp.err
python -c "
import json; j=json.load(open('gpurun_out/bp.json'));print(j['next_rows'])"
