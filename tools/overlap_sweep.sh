# step time: 1 vs 2 vs 4 CUDA streams, alternated (measurement)
run() { python bench.py --steps 20 --warmup 3 --no-n1 --no-cpu-baseline --no-e2e "$@" 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), d['config']['streams'])"; }
for i in 1 2 3; do
echo "s1 $(run)"
echo "s2 $(run --streams 2)"
echo "s4 $(run --streams 4)"
done
