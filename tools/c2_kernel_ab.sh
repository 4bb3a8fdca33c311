# A/B of alternate library builds (tools/libmasq_<tag>.so) on the c2 step: step time and the
# weight-side kernels; restores the first tag's build last
out=gpurun_out/c2_kernel_ab.txt
: > $out
for rep in 1 2 3; do
  for tag in "$@"; do
    cp tools/libmasq_$tag.so paper_2603_04800_b200/libmasq.so
    r=$(timeout 300 python bench.py --workload c2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-n1 | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],4), {k: round(v["ms_per_step"],4) for k,v in d["kernels"].items() if k in ("wcolmax","wquant","init","wscale","stats","aquant")})')
    echo "$tag c2 $r" >> $out
  done
done
cp tools/libmasq_$1.so paper_2603_04800_b200/libmasq.so
cat $out
