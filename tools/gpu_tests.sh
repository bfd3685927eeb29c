#!/bin/bash
# GPU test suite with the parity log (run on the box via gpurun): results under gpurun_out/$1
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-tests}; mkdir -p $O
export GS_PARITY_LOG=$O/parity_stats.jsonl
rm -f $GS_PARITY_LOG
timeout 1500 python -m pytest tests -m gpu -q -rf --durations=15 ${@:2} > $O/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -30 $O/pytest_gpu.log
