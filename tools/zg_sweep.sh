# CMC first factor at T = 16384, d = 3584: split-K count x ring stages (measurement)
for cfg in "0 0" "2 3" "2 4" "0 0" "2 3"; do
  set -- $cfg
  echo "splits=$1 stages=$2 $(MASQ_ZGEMM_SPLITS=$1 MASQ_ZGEMM_STAGES=$2 python tools/gemm_bench.py --n 3584 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["fwd_r64"].get("zgemm"), d["fwd_r64"].get("zcombine"))')"
done
