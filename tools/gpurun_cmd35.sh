cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_server.py tests/test_gpu_gate.py tests/test_gpu_workers.py tests/test_gpu_dropin_reference.py -q 2>&1 | tail -5 > gpurun_out/r2_t35.log
timeout 120 python tools/percall_probe.py > gpurun_out/r2_percall_py2.txt 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > gpurun_out/r2_bench_default2.json 2> gpurun_out/r2_bench_default2.err
