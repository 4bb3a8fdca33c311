# per-kernel CUDA-event times of the c3 step with and without programmatic dependent launch
out=gpurun_out/pdl_kernel_ab.txt
: > $out
for v in 1 0 1 0 1 0; do
  r=$(MASQ_PDL=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-n1 | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],3), "unprof", round(d["unprofiled"]["ms_per_step"],3), {k: round(v["ms_per_step"],3) for k,v in d["kernels"].items() if k in ("gemm_ref","gemm_fwd","gemm_loss","aquant","stats","wquant","zgemm")}, d["clocks"]["sm_mhz"])')
  echo "pdl=$v $r" >> $out
done
cat $out
