# c3 step: the activation quantizer's chunks per thread (MASQ_AQ_CPL) and the CMC first factor's
# split / pair / stage knobs, per-kernel ms per step (measurement helper)
out=gpurun_out/hbm_knob_sweep.txt
: > $out
run() {
  echo "$1 $(env $1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-n1 | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d["kernels"]; print(round(d["ms_per_step"],3), {n: (round(k[n]["ms_per_step"],3), round(k[n].get("frac",0),2)) for n in ("aquant","zgemm","wquant","wcolmax","stats","init")})')" >> $out
}
run "MASQ_NONE=1"
for c in 2 3 4 5 6; do run "MASQ_AQ_CPL=$c"; done
run "MASQ_ZGEMM_PAIR=0"
run "MASQ_ZGEMM_PAIR=0 MASQ_ZGEMM_SPLITS=2"
run "MASQ_ZGEMM_PAIR=0 MASQ_ZGEMM_SPLITS=4"
run "MASQ_ZGEMM_STAGES=2"
cat $out
