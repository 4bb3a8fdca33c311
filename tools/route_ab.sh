# routing: single-CTA route_kernel (MASQ_ROUTE_V1=1, + perm memset) vs the two-pass multi-CTA routing
out=gpurun_out/route_ab.txt
: > $out
for rep in 1 2; do
  for v in 0 1; do
    for wl in c2 c3; do
      if [ $v = 1 ]; then export MASQ_ROUTE_V1=1; else unset MASQ_ROUTE_V1; fi
      r=$(timeout 300 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-n1 | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],4), "route", round(d["kernels"]["route"]["ms_per_step"],4), "bd", d["kernels_source"][-22:], "clk", d["clocks"]["sm_mhz"])')
      echo "v1=$v $wl $r" >> $out
    done
  done
done
unset MASQ_ROUTE_V1
cat $out
