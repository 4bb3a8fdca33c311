# A/B of alternate library builds (tools/libmasq_<tag>.so) on the c2 and c3 steps (profiled,
# unprofiled and 2-stream timings); restores the first tag's build last
out=gpurun_out/step_ab.txt
: > $out
for rep in 1 2; do
  for tag in "$@"; do
    cp tools/libmasq_$tag.so paper_2603_04800_b200/libmasq.so
    for wl in c2 c3; do
      r=$(timeout 300 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-n1 | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],4), "unprof", round(d["unprofiled"]["ms_per_step"],4), "2st", round(d["overlapped"]["ms_per_step"],4), "clk", d["clocks"]["sm_mhz"])')
      echo "$tag $wl $r" >> $out
    done
  done
done
cp tools/libmasq_$1.so paper_2603_04800_b200/libmasq.so
cat $out
