for v in sep in sep in; do
  if [ $v = sep ]; then MASQ_SEPARATE_INV=1 C5_KMAX=3 python tools/sweep_c5.py > /tmp/c5.log 2>&1; else C5_KMAX=3 python tools/sweep_c5.py > /tmp/c5.log 2>&1; fi
  echo "$v $(python -c '
import json
out=[]
for l in open("/tmp/c5.log"):
  if l.startswith("{\"T\""):
    r=json.loads(l); out.append((r["n"],r["r"],r["T"],round(r["call_ms"]*1e3,1)))
print(out)')"
done
