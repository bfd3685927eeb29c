cd $GRAFT_REPO_ROOT
O=gpurun_out/r2f; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rasterize_warp -c 1 -o $O/full_rw_C4x16 python bench.py --views 16 --profile-steps 1 --no-e2e --no-cpu-baseline > $O/ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rasterize_warp -c 1 -o $O/full_rw_C5x4 python bench.py --config C5 --views 4 --profile-steps 1 --no-e2e --no-cpu-baseline > $O/ncu2.log 2>&1
timeout 900 env GS_RASTER_LEGACY=1 ncu --set full --clock-control none --import-source on -k regex:rasterize_kernel -c 1 -o $O/full_rl_C5x4 python bench.py --config C5 --views 4 --profile-steps 1 --no-e2e --no-cpu-baseline > $O/ncu3.log 2>&1
ls -la $O
