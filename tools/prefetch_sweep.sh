# f1 sweep (tools/prefetch_bench.py): pool budgets below and above the per-pass working set, both
# prefetch policies, decode and prefill, HBM-resident and host-offload masters.
mkdir -p gpurun_out/pf
for cfg in "--layers 8 --passes 4 --budget 0.15" "--layers 8 --passes 4 --budget 0.25" \
           "--prefill --layers 8 --passes 2 --budget 0.2" "--prefill --layers 8 --passes 2 --budget 0.3" \
           "--offload --layers 4 --passes 3 --budget 0.15" "--offload --prefill --layers 4 --passes 2 --budget 0.2"; do
  for pol in critical tiered; do
    name=$(echo "$cfg $pol" | tr -c 'a-z0-9.' '_')
    timeout 600 python tools/prefetch_bench.py $cfg --policy $pol 2>/dev/null | tail -1 > gpurun_out/pf/$name.json
    python - "$cfg $pol" gpurun_out/pf/$name.json <<'PY'
import json, sys
try:
    j = json.load(open(sys.argv[2]))
except Exception as e:
    print(sys.argv[1], "FAILED", e); sys.exit()
o = j.get("overlap", {}); h = j.get("overlap_h2d", {})
side = [v for v in o.get("per_stream", {}).values() if v["role"].startswith("side")]
print(sys.argv[1], "| demand %.2f ms (misses %d) | prefetch %.2f ms (misses %d, prefetched %d, hits-from-prefetch %d, evictions %d) | side quantize hidden %.2f | ffn with copy in flight %s" % (
    j["demand_only"]["ms_per_pass"], j["demand_only"]["stats"]["misses"], j["prefetch"]["ms_per_pass"],
    j["prefetch"]["stats"]["misses"], j["prefetch"]["stats"]["prefetched"], j["prefetch"]["stats"]["prefetch_hits"],
    j["prefetch"]["stats"]["evictions"], side[0]["frac_hidden"] if side else 0,
    h.get("frac_of_ffn_time_with_a_prefetch_copy_in_flight")))
PY
  done
done
