cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke59.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -5 > gpurun_out/r2_gpu_all59.log
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_b59.json 2> gpurun_out/r2_b59.err
