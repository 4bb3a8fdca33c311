# raster of the X.W GEMM at the deep-K down shape and gate_up: n-grouped (g > 0) vs m-grouped (g < 0)
for shape in "18944 3584" "3584 37888"; do
for g in 16 -2 -4 -8 -16; do
  t=$(MASQ_RASTER_GROUP=$g python tools/refgemm.py $shape 16384 10 2>&1)
  b=$(MASQ_RASTER_GROUP=$g timeout 120 ncu --metrics dram__bytes_read.sum --clock-control none -k regex:masq_gemm -s 2 -c 1 --csv python tools/refgemm.py $shape 16384 1 2>/dev/null | grep dram__bytes_read | awk -F'","' '{print $NF}')
  echo "$t read=$b"
done; done
