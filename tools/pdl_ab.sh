# N3 decode call with / without programmatic dependent launch of the decode kernel (measurement)
for v in 0 1 0 1; do
  MASQ_DECODE_PDL=$v python tools/decode_bench.py > /dev/null 2>&1
  echo "pdl=$v $(python -c 'import json; d=json.load(open("gpurun_out/decode_bench.json")); print({k: round(v["graph_call_ms"]*1e3,1) for k,v in d.items() if isinstance(v, dict)})')"
done
