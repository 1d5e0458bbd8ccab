set -u
O=gpurun_out/r02; mkdir -p $O
NCU="ncu --set full --clock-control none --import-source on -f"
for w in prefill finegrained; do
  python tools/profile_step.py --workload $w > $O/step_$w.json 2>/dev/null
  $NCU -k regex:k_prefill_gemm -s 4 -c 2 -o $O/$w python tools/profile_step.py --workload $w > $O/ncu_$w.log 2>&1
  python tools/ncu_summary.py $O/$w.ncu-rep $O/step_$w.json > $O/ncu_$w.md 2>/dev/null
done
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_|gemv|gemm" -c 3000 --csv \
    --log-file $O/launches_prefill.csv python bench.py --workload prefill --steps 4 --warmup 3 --copies 1 --no-cpu-baseline > /dev/null 2>&1
python tools/launch_shares.py $O/launches_prefill.csv > $O/launch_shares_prefill.md
head -12 $O/launch_shares_prefill.md
