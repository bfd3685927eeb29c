cd $GRAFT_REPO_ROOT
O=gpurun_out/r2w; mkdir -p $O
bash tools/var_bench.sh cur ch1 ch4 > $O/var.txt 2>&1
grep -v "^\[gs\]" $O/var.txt
