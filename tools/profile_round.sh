#!/bin/bash
# Round profile capture (run on the GPU box via gpurun): the bench line, the ncu
# launch list of the same command, DRAM traffic of gs_rasterize, and --set full
# captures of the raster (16-view subset) and the N2 / bin-sort kernels.
set -x
cd $GRAFT_REPO_ROOT
O=gpurun_out/r1e; mkdir -p $O
timeout 600 python bench.py --steps 10 --warmup 3 --n2 --refine 32 > $O/bench_C4.json 2> $O/bench_C4.err || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C4.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_launch.log 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:^rasterize -c 1 --csv --log-file $O/dram_raster_C4.csv python bench.py --steps 1 --warmup 3 --profile-steps 1 --no-e2e --no-cpu-baseline > $O/ncu_dram.log 2>&1
if [ "$1" == "full" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:^rasterize -c 1 -o $O/full_raster_C4x16 python bench.py --views 16 --profile-steps 1 --no-e2e --no-cpu-baseline > $O/ncu_full_r.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"row_kernel|fine_kernel|count_kernel|scatter_kernel|warp_sort|pnp_kernel|project_kernel" -c 8 -o $O/full_match_bin python bench.py --views 16 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --n2 --n2-pairs 8 > $O/ncu_full_m.log 2>&1
fi
ls -la $O
