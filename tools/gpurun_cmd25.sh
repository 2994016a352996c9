cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_sharded.py -q -k torch_workers 2>&1 | tail -5 > gpurun_out/r2_t25.log
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > gpurun_out/r2_bench_default.json 2> gpurun_out/r2_bench_default.err
