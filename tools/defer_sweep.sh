# forward GEMM with CMC (r = 64): where in the next unit's k-block stream the CMC MMAs go
for dv in 4 16 20 24 27; do
  echo "gate defer=$dv $(MASQ_CMC_DEFER=$dv python tools/gemm_bench.py | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["fwd_r0_gemm_tops"]), round(d["fwd_r64_gemm_tops"]), d["fwd_r64"]["gemm_fwd"])')"
  echo "o    defer=$dv $(MASQ_CMC_DEFER=$dv python tools/gemm_bench.py --n 3584 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["fwd_r0_gemm_tops"]), round(d["fwd_r64_gemm_tops"]), d["fwd_r64"]["gemm_fwd"])')"
  echo "down defer=$dv $(MASQ_CMC_DEFER=$dv python tools/gemm_bench.py --d 18944 --n 3584 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["fwd_r0_gemm_tops"]), round(d["fwd_r64_gemm_tops"]), d["fwd_r64"]["gemm_fwd"])')"
done
