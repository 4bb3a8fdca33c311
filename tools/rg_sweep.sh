for shape in "3584 37888" "18944 3584"; do
for g in 2 4 8 16 32; do
  MASQ_RASTER_GROUP=$g python tools/refgemm.py $shape 16384 10 >> gpurun_out/rg_time.txt 2>&1
  MASQ_RASTER_GROUP=$g timeout 120 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum --clock-control none -k regex:masq_gemm -s 2 -c 1 --csv python tools/refgemm.py $shape 16384 1 > gpurun_out/rg_${g}_${shape// /_}.csv 2>&1
done; done
