# activation quantizer chunks per thread (MASQ_AQ_CPL) at small T: c5 call / aquant kernel times
out=gpurun_out/aqcpl_ab.txt
: > $out
for rep in 1 2; do
  for v in 8 4 2; do
    MASQ_AQ_CPL=$v C5_KMAX=4 timeout 600 python tools/sweep_c5.py 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("cpl='$v'", [(x["T"], x["n"], x["r"], round(x["call_ms"]*1e3,1), round(x["kernels_ms"]["aquant"]*1e3,1)) for x in d["c5_sweep"] if x["n"] == 3584])' >> $out
  done
done
cat $out
