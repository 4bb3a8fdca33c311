# A/B of alternate library builds tools/libmasq_<tag>.so on the bench step's kernel table (measurement helper)
for tag in "$@"; do
  cp tools/libmasq_$tag.so paper_2603_04800_b200/libmasq.so
  echo "$tag $(python bench.py --steps 10 --warmup 3 --no-n1 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3), {k: round(v["ms_per_step"],3) for k,v in d["kernels"].items() if k in ("wcolmax","wquant","aquant","stats")})')"
done
