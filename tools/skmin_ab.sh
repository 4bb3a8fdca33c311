# stream-K remainder at shallow K (MASQ_SK_MINKB=16) vs the default deep-K-only threshold (64)
out=gpurun_out/skmin_ab.txt
: > $out
for rep in 1 2; do
  for v in 64 16; do
    export MASQ_SK_MINKB=$v
    C5_KMAX=3 timeout 600 python tools/sweep_c5.py 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("minkb='$v' c5", [(x["T"], x["n"], x["r"], round(x["call_ms"]*1e3,1), round(x["gemm_ms"]*1e3,1)) for x in d["c5_sweep"]])' >> $out
    for wl in c2 c3; do
      r=$(timeout 300 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-n1 | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],4), {k: round(v["ms_per_step"],4) for k,v in d["kernels"].items() if k.startswith("gemm")}, "clk", d["clocks"]["sm_mhz"])')
      echo "minkb=$v $wl $r" >> $out
    done
  done
done
unset MASQ_SK_MINKB
cat $out
