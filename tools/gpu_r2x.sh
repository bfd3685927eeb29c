cd $GRAFT_REPO_ROOT
O=gpurun_out/r2x; mkdir -p $O
bash tools/var_bench.sh cur hionly > $O/var.txt 2>&1
grep -v "^\[gs\]" $O/var.txt
