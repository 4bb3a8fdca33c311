# stream-K remainder on / off (MASQ_STREAMK) at c3 / c5 shapes: GEMM kernel ms (tools/gemm_bench.py)
out=gpurun_out/sk_ab.txt
: > $out
for shape in "--T 4096 --n 3584" "--T 16384 --n 3584" "--T 16384 --n 4608" "--T 4096 --d 18944 --n 3584" "--T 16384 --d 18944 --n 3584" "--T 2048 --n 3584" "--T 8192 --n 3584"; do
  for sk in 1 0; do
    echo "SK=$sk $shape $(MASQ_STREAMK=$sk timeout 120 python tools/gemm_bench.py $shape | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print({k: round(v["gemm_fwd" if "fwd" in k else "gemm_"+k]*1000,1) for k,v in d.items() if k in ("fwd_r0","fwd_r64","acc","ref")})')" >> $out
  done
done
cat $out
