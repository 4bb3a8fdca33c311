# CMC first factor at T = 16384: cluster-pair split-K vs one CTA per tile (MASQ_ZGEMM_PAIR=0), alternated
for i in 1 2; do
  for v in 0 1; do
    echo "pair=$v gate $(MASQ_ZGEMM_PAIR=$v python tools/gemm_bench.py | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["fwd_r64"].get("zgemm"))')  down $(MASQ_ZGEMM_PAIR=$v python tools/gemm_bench.py --d 18944 --n 3584 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["fwd_r64"].get("zgemm"))')"
  done
done
