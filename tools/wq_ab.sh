run() { python bench.py --steps 10 --warmup 3 --no-n1 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3), {k: round(v["ms_per_step"],3) for k,v in d["kernels"].items() if k in ("wcolmax","wquant")})'; }
for i in 1 2; do
cp tools/libmasq_wq2.so paper_2603_04800_b200/libmasq.so
echo "v1  $(MASQ_WQUANT_V1=1 run)"
echo "wq2 $(run)"
cp tools/libmasq_wq3.so paper_2603_04800_b200/libmasq.so
echo "wq3 $(run)"
done
cp tools/libmasq_wq2.so paper_2603_04800_b200/libmasq.so
