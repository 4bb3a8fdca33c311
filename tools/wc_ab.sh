# weight column maxima: TMA-fed kernel vs the strip kernel (MASQ_WCOLMAX_V1), alternated (measurement)
run() { python bench.py --steps 10 --warmup 3 --no-n1 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3), {k: round(v["ms_per_step"],3) for k,v in d["kernels"].items() if k in ("wcolmax","wquant")})'; }
for i in 1 2; do echo "v1  $(MASQ_WCOLMAX_V1=1 run)"; echo "tma $(run)"; done
