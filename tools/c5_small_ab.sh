# A/B of alternate library builds (tools/libmasq_<tag>.so) on the c5 forward call at 1k-4k tokens
# (whole-call time, profiler off); restores the first tag's build last
out=gpurun_out/c5_small_ab.txt
: > $out
for rep in 1 2; do
  for tag in "$@"; do
    cp tools/libmasq_$tag.so paper_2603_04800_b200/libmasq.so
    C5_KMAX=3 timeout 600 python tools/sweep_c5.py 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("'$tag'", [(x["T"], x["n"], x["r"], round(x["call_ms"]*1e3,1)) for x in d["c5_sweep"]])' >> $out
  done
done
cp tools/libmasq_$1.so paper_2603_04800_b200/libmasq.so
cat $out
