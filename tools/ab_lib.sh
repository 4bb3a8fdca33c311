# A/B of alternate library builds tools/libmasq_<tag>.so on tools/kbench.py (measurement helper)
for tag in "$@"; do
  cp tools/libmasq_$tag.so paper_2603_04800_b200/libmasq.so
  echo "$tag $(python tools/kbench.py | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print({k:(round(v["wq1"]["wcolmax"],4), round(v["wq2_ms"],4), round(v["stats_ms"],4)) for k,v in d.items()})')"
done
