# activation quantizer chunks per thread (MASQ_AQ_CPL 8 = default vs 4) on the c2 / c3 steps
out=gpurun_out/aqcpl_step_ab.txt
: > $out
for rep in 1 2 3; do
  for v in 8 4; do
    for wl in c2 c3; do
      r=$(MASQ_AQ_CPL=$v timeout 300 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-n1 | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],4), "med", round(d["ms_per_step_median"],4), "aquant", round(d["kernels"]["aquant"]["ms_per_step"],4), "clk", d["clocks"]["sm_mhz"])')
      echo "cpl=$v $wl $r" >> $out
    done
  done
done
cat $out
