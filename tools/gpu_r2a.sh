cd $GRAFT_REPO_ROOT
O=gpurun_out/r2a; mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/ex2_probe.cu -o /tmp/ex2_probe && timeout 120 /tmp/ex2_probe > $O/ex2_probe.json 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 > $O/bench_C4.json 2> $O/bench_C4.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:^rasterize -c 1 -o $O/full_raster_C4x16 python bench.py --views 16 --profile-steps 1 --no-e2e --no-cpu-baseline > $O/ncu_full_r.log 2>&1
ls -la $O
