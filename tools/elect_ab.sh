# after the warp-wide MMA / TMA issue loops: GEMM rates at the four c3 linears (raster: fixed
# 16-n-tile groups vs the 32 MB L2 budget), the N3 prefill GEMM, the N2 Gram and the c3 step
out=gpurun_out/elect_ab.txt
: > $out
for shape in "3584 4608" "3584 3584" "3584 37888" "18944 3584"; do
  set -- $shape
  for cfg in "MASQ_RASTER_GROUP=16" "MASQ_RASTER_L2MB=32"; do
    r=$(env $cfg timeout 120 python tools/gemm_bench.py --d $1 --n $2 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print({k: round(v) for k,v in d.items() if k in ("fwd_r0_gemm_tops","fwd_r64_gemm_tops","acc_gemm_tops","ref_tflops","cublas_int_mm_tops","cublas_bf16_tflops")})')
    echo "d=$1 n=$2 $cfg $r" >> $out
  done
done
timeout 300 python tools/w4g_bench.py 16384 > gpurun_out/w4g_elect.log 2>&1; grep -o '"gemm_tops": [0-9.]*' gpurun_out/w4g_elect.log >> $out
timeout 300 python tools/cmc_bench.py qkv,down > gpurun_out/cmc_elect.log 2>&1; grep -o '"gram_ms": [0-9.]*' gpurun_out/cmc_elect.log >> $out
for i in 1 2; do
  echo "bench $(timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-n1 | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],3), {k: round(v["ms_per_step"],3) for k,v in d["kernels"].items()})')" >> $out
done
cat $out
