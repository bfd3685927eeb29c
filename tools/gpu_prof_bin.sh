cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-pb}; mkdir -p $O
for k in project_kernel count_kernel scatter_kernel warp_sort_kernel; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 2 --launch-count 1 -o $O/${k}_C4x16 python bench.py --views 16 --profile-steps 1 --no-e2e --no-cpu-baseline > $O/ncu_$k.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 2 --launch-count 1 -o $O/${k}_C5x8 python bench.py --config C5 --views 8 --profile-steps 1 --no-e2e --no-cpu-baseline > $O/ncu5_$k.log 2>&1
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C5.csv python bench.py --config C5 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/launch5.log 2>&1
ls -la $O
