cd $GRAFT_REPO_ROOT
O=gpurun_out/r2r; mkdir -p $O
bash tools/var_bench.sh main se64n4 se64n5 > $O/var.txt 2>&1
cat $O/var.txt
GS_LIB=$GRAFT_REPO_ROOT/paper_2507_15683_b200/_build/var_se64n5/libgs.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > $O/pytest_se64n5.log 2>&1; echo "rc=$?" >> $O/pytest_se64n5.log
tail -n 2 $O/pytest_se64n5.log
