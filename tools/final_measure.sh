# end-of-session measurement set (1 GPU): c3 / c2 bench lines, the ncu launch list of the c3 step,
# per-kernel DRAM traffic (profiles/ncu_traffic.json input); $1 = file tag (default r02c)
tag=${1:-r02c}
set -x
timeout 600 python bench.py > gpurun_out/bench_c3.log 2>&1; tail -1 gpurun_out/bench_c3.log > gpurun_out/bench_c3.json
timeout 600 python bench.py --workload c2 > gpurun_out/bench_c2.log 2>&1; tail -1 gpurun_out/bench_c2.log > gpurun_out/bench_c2.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$tag.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-n1 > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python bench.py --profile-only > gpurun_out/traffic_$tag.csv 2>gpurun_out/traffic_$tag.err
python tools/traffic_json.py gpurun_out/traffic_$tag.csv gpurun_out/ncu_traffic_$tag.json > /dev/null
python -c "import json; d=json.load(open('gpurun_out/bench_c3.json')); print(d['value'], d['ms_per_step'], d['roofline'], d['clocks'])"
python -c "import json; d=json.load(open('gpurun_out/bench_c2.json')); print(d['value'], d['ms_per_step'], d['roofline'])"
