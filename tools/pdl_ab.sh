# N3 decode call: previous (memset + inverse factors + quantizer, MASQ_AQUANT_V1) vs the one-launch
# quantizer, both with programmatic dependent launch of the decode kernel (measurement)
for v in 1 0 1 0; do
  if [ $v = 1 ]; then MASQ_AQUANT_V1=1 python tools/decode_bench.py > /dev/null 2>&1; else python tools/decode_bench.py > /dev/null 2>&1; fi
  echo "aquant_v1=$v $(python -c 'import json; d=json.load(open("gpurun_out/decode_bench.json")); print({k: round(v["graph_call_ms"]*1e3,1) for k,v in d.items() if isinstance(v, dict)})')"
done
