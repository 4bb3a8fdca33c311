# programmatic dependent launch across the library's kernels (MASQ_PDL=1, default) vs plain stream
# serialisation (MASQ_PDL=0): c3 and c2 steps (profiled region, unprofiled region, 2 streams) and
# the c5 forward call at 1k-8k tokens (whole-call time, profiler off)
out=gpurun_out/pdl_step_ab.txt
: > $out
for v in 1 0 1 0; do
  for wl in c3 c2; do
    r=$(MASQ_PDL=$v timeout 300 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-n1 | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],4), "unprof", round(d["unprofiled"]["ms_per_step"],4), "2st", round(d["overlapped"]["ms_per_step"],4), "clk", d["clocks"]["sm_mhz"])')
    echo "pdl=$v $wl $r" >> $out
  done
  MASQ_PDL=$v C5_KMAX=4 timeout 600 python tools/sweep_c5.py 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("pdl='$v' c5", [(x["T"], x["n"], x["r"], round(x["call_ms"]*1e3,1)) for x in d["c5_sweep"]])' >> $out
done
cat $out
