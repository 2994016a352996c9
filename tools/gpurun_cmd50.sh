cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_replay.py tests/test_boundary.py -q -x 2>&1 | tail -3 > gpurun_out/r2_t50.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_b50.json 2> gpurun_out/r2_b50.err
