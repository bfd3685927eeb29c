cd $GRAFT_REPO_ROOT
O=gpurun_out/dbg; mkdir -p $O
export CUDA_LAUNCH_BLOCKING=1
for v in f1 f2 main; do
  if [ "$v" == "main" ]; then L=paper_2507_15683_b200/libgs.so; else L=paper_2507_15683_b200/_build/var_$v/libgs.so; fi
  GS_LIB=$L timeout 300 python bench.py --config C4 --scale 0.02 --views 16 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/$v.log 2>&1; echo "$v rc=$?"
  grep -m2 "illegal\|GS_CHECK\|ms_per_step" $O/$v.log | cut -c1-200
done
