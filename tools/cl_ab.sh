# A/B of the GEMM cluster size (MASQ_GEMM_CL = 2 | 4) on tools/gemm_bench.py shapes and the c3 bench step
# (measurement helper)
out=gpurun_out/cl_ab.txt
: > $out
for shape in "--n 18944" "--n 3584" "--n 4608" "--d 18944 --n 3584"; do
  for cl in 2 4; do
    echo "CL=$cl $shape $(MASQ_GEMM_CL=$cl timeout 120 python tools/gemm_bench.py $shape | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print({k: round(v) for k,v in d.items() if k.endswith("_tops") or k.endswith("tflops")})')" >> $out
  done
done
for cl in 2 4 2 4; do
  echo "CL=$cl bench $(MASQ_GEMM_CL=$cl timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-n1 | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],3), {k: round(v["ms_per_step"],3) for k,v in d["kernels"].items() if k.startswith("gemm")})')" >> $out
done
cat $out
