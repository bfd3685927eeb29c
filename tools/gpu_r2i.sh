cd $GRAFT_REPO_ROOT
O=gpurun_out/r2i; mkdir -p $O
for k in count_kernel scatter_kernel; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 2 --launch-count 1 -o $O/${k}_C4x16 python bench.py --views 16 --profile-steps 1 --no-e2e --no-cpu-baseline > $O/ncu_$k.log 2>&1
done
bash tools/gpu_sanitize.sh r2i_san
