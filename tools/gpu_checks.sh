cd $GRAFT_REPO_ROOT
# the GPU suite and the sanitize case on the GS_CHECKS build (device-side bounds checks)
O=gpurun_out/checks; mkdir -p $O
export GS_LIB=paper_2507_15683_b200/_build/checks/libgs.so
{ echo "# GS_CHECKS build (tools/build_checks.sh: device-side bounds checks, -DGS_CHECKS) on the B200 -- round 2, final kernels"
  echo "## tools/sanitize_case.py"; timeout 300 python tools/sanitize_case.py 2>&1 | tail -2; echo "rc=$?"
  echo "## python -m pytest tests -m gpu (GS_LIB = the checked build)"; timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -3; echo "rc=$?"
  echo "## bench C4 (checked build, 2 steps)"; timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | cut -c1-120; echo "rc=$?"
} > $O/bounds_checks.txt 2>&1
cat $O/bounds_checks.txt
