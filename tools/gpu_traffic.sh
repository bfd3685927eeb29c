cd $GRAFT_REPO_ROOT
# DRAM traffic + issue activity of one gs_rasterize launch in the bench's launch configuration
O=gpurun_out/traffic; mkdir -p $O
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,smsp__thread_inst_executed.sum
timeout 900 ncu --metrics $M --clock-control none --csv -k regex:^rasterize -s 4 -c 1 --log-file $O/raster_C4.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/c4.log 2>&1
timeout 900 ncu --metrics $M --clock-control none --csv -k regex:^rasterize -s 4 -c 1 --log-file $O/raster_C5.csv python bench.py --config C5 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/c5.log 2>&1
cat $O/raster_C4.csv $O/raster_C5.csv | grep -v "^==" | cut -c1-400
