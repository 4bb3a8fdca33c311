# A/B of alternate library builds tools/libmasq_<tag>.so on tools/gemm_bench.py (measurement helper)
for tag in "$@"; do
  cp tools/libmasq_$tag.so paper_2603_04800_b200/libmasq.so
  echo "$tag gate $(python tools/gemm_bench.py | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print({k: round(v) for k,v in d.items() if k.endswith("_tops") or k.endswith("tflops")})')"
  echo "$tag o    $(python tools/gemm_bench.py --n 3584 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print({k: round(v) for k,v in d.items() if k.endswith("_tops") or k.endswith("tflops")})')"
done
