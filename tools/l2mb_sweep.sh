# raster group sized by an L2 budget (MASQ_RASTER_L2MB) vs the fixed 16-n-tile group (MASQ_RASTER_GROUP=16):
# GEMM rates (tools/gemm_bench.py) and the X.W GEMM's DRAM reads (ncu) at the four c3 linears
out=gpurun_out/l2mb_sweep.txt
: > $out
for shape in "3584 4608" "3584 3584" "3584 37888" "18944 3584"; do
  set -- $shape
  for cfg in "MASQ_RASTER_GROUP=16" "MASQ_RASTER_L2MB=32" "MASQ_RASTER_L2MB=64" "MASQ_RASTER_L2MB=96"; do
    r=$(env $cfg timeout 120 python tools/gemm_bench.py --d $1 --n $2 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print({k: round(v) for k,v in d.items() if k in ("fwd_r64_gemm_tops","acc_gemm_tops","ref_tflops")})')
    b=$(env $cfg timeout 120 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:masq_gemm -s 2 -c 1 --csv python tools/refgemm.py $1 $2 16384 1 2>/dev/null | grep dram__bytes | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ')
    echo "d=$1 n=$2 $cfg $r ref_dram_rw=$b" >> $out
  done
done
cat $out
