cd $GRAFT_REPO_ROOT
O=gpurun_out/r2q; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_n4.py -q -k "joint or radiance or training" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -n 3 $O/pytest.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --n4 > $O/bench_C4_n4.json 2> $O/bench_C4_n4.err
python -c "import json; d=json.loads(open('$O/bench_C4_n4.json').read().strip().splitlines()[-1]); print(d['n4'])"
