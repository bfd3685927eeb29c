cd $GRAFT_REPO_ROOT
# ncu --set full of the projection, count and class-sort kernels after the round-2 changes (C4x16, C5x8)
O=gpurun_out/r2p; mkdir -p $O
for k in project_kernel count_kernel class_sort_kernel; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 2 --launch-count 1 -o $O/${k}_C4x16 python bench.py --views 16 --profile-steps 1 --no-e2e --no-cpu-baseline > $O/ncu_$k.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:project_kernel --launch-skip 2 --launch-count 1 -o $O/project_kernel_C5x8 python bench.py --config C5 --views 8 --profile-steps 1 --no-e2e --no-cpu-baseline > $O/ncu5_project.log 2>&1
ls -la $O
