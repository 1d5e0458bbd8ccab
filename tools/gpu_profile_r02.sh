# Round-2 evidence (run from the repo root on a B200): ncu --set full captures of the dominant
# kernels (decode GEMV of the bench's layer-20 step, prefill grouped GEMM, fine-grained decode /
# prefill, f3 attention mass), each summarised against the step's algorithmic work, and the
# launch list of the default bench command (per-kernel share of the step).  Outputs under
# gpurun_out/r02/.
set -u
O=gpurun_out/r02
mkdir -p $O
NCU="ncu --set full --clock-control none --import-source on -f"
for w in decode prefill finegrained_decode finegrained; do
  python tools/profile_step.py --workload $w > $O/step_$w.json 2>/dev/null
  k=k_decode_gemv; case $w in prefill|finegrained) k=k_prefill_gemm;; esac
  $NCU -k regex:$k -s 4 -c 2 -o $O/$w python tools/profile_step.py --workload $w > $O/ncu_$w.log 2>&1
  python tools/ncu_summary.py $O/$w.ncu-rep $O/step_$w.json > $O/ncu_$w.md 2>/dev/null
  tail -n 1 $O/ncu_$w.log
done
$NCU -k regex:k_attn_mass -c 2 -o $O/attn python tools/attn_probe.py 2048 > $O/ncu_attn.log 2>&1
python tools/ncu_summary.py $O/attn.ncu-rep > $O/ncu_attn.md 2>/dev/null
# launch list of the bench command (kernels of this library only; per-launch, serialised, cold)
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_|gemv|gemm" -c 3000 --csv \
    --log-file $O/launches_decode.csv python bench.py --steps 8 --warmup 3 --copies 1 --no-cpu-baseline --main-only > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_|gemv|gemm" -c 3000 --csv \
    --log-file $O/launches_prefill.csv python bench.py --workload prefill --steps 4 --warmup 3 --copies 1 --no-cpu-baseline > /dev/null 2>&1
for f in decode prefill; do python tools/launch_shares.py $O/launches_$f.csv > $O/launch_shares_$f.md; done
ls -la $O | head -40
