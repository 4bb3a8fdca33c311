# X.W GEMM L2 hints (MASQ_REF_POLICY: bit 0 A evict_first, bit 1 B evict_last): time + DRAM reads
out=gpurun_out/refpol_sweep.txt
: > $out
for shape in "3584 37888" "18944 3584" "3584 4608"; do
  set -- $shape
  for pol in 3 2 1 0; do
    t=$(MASQ_REF_POLICY=$pol python tools/refgemm.py $1 $2 16384 10 2>&1 | tail -1)
    b=$(MASQ_REF_POLICY=$pol timeout 120 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:masq_gemm -s 2 -c 1 --csv python tools/refgemm.py $1 $2 16384 1 2>/dev/null | grep dram__bytes | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ')
    echo "pol=$pol $t dram_rw=$b" >> $out
  done
done
cat $out
