# A1 stats: minimum rows per strip (MASQ_STATS_MINROWS, default 64) on the c2 / c3 steps
out=gpurun_out/stats_rows_ab.txt
: > $out
for rep in 1 2; do
  for v in 64 32 16; do
    for wl in c2 c3; do
      r=$(MASQ_STATS_MINROWS=$v timeout 300 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-n1 | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],4), "med", round(d["ms_per_step_median"],4), "stats", round(d["kernels"]["stats"]["ms_per_step"],4), "clk", d["clocks"]["sm_mhz"])')
      echo "minrows=$v $wl $r" >> $out
    done
  done
done
cat $out
