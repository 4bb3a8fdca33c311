# CMC first factor split count at small T (MASQ_ZGEMM_SPLITS; 0 = default rule) on the c5 r=64 call
out=gpurun_out/zsplit_ab.txt
: > $out
for rep in 1 2; do
  for v in 0 2 4 8; do
    MASQ_ZGEMM_SPLITS=$v C5_KMAX=4 timeout 600 python tools/sweep_c5.py 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("splits='$v'", [(x["T"], x["n"], round(x["call_ms"]*1e3,1), round(x["kernels_ms"].get("zgemm",0)*1e3,1), round(x["kernels_ms"].get("zcombine",0)*1e3,1)) for x in d["c5_sweep"] if x["r"] == 64 and x["n"] == 3584])' >> $out
  done
done
cat $out
