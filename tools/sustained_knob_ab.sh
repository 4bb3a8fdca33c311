# c3 step in the sustained (power-capped) regime: GEMM raster / L2-policy knobs, alternated
out=gpurun_out/sustained_knob_ab.txt
: > $out
for rep in 1 2; do
  for cfg in ${CFGS:-"X=0" "MASQ_RASTER_L2MB=16" "MASQ_RASTER_L2MB=64" "MASQ_REF_POLICY=3" "MASQ_I8_POLICY=3"}; do
    r=$(env $cfg timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-n1 | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],3), "med", round(d["ms_per_step_median"],3), {k: round(v["ms_per_step"],3) for k,v in d["kernels"].items() if k.startswith("gemm")}, d["clocks"]["sm_mhz"], d["clocks"]["sm_min_mhz"], d["clocks"]["reasons"])')
    echo "$cfg $r" >> $out
  done
done
cat $out
