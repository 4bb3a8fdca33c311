# int8 GEMM L2 hints (MASQ_I8_POLICY: bit 0 A evict_first, bit 1 B evict_last): forward GEMM ms
out=gpurun_out/i8pol_sweep.txt
: > $out
for shape in "--n 37888" "--d 18944 --n 3584" "--n 4608" "--n 3584"; do
  for pol in 0 1 2 3; do
    echo "pol=$pol $shape $(MASQ_I8_POLICY=$pol timeout 120 python tools/gemm_bench.py $shape | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print({k: round(v["gemm_fwd" if "fwd" in k else "gemm_"+k]*1000,1) for k,v in d.items() if k in ("fwd_r0","fwd_r64","acc")})')" >> $out
  done
done
cat $out
