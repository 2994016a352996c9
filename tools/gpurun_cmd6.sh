cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_freerun.py -q 2>&1 | tail -30 > gpurun_out/r2_t6.log
(time timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29514 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/r2_bench_n4.json 2> gpurun_out/r2_bench_n4.err) 2> gpurun_out/r2_bench_n4.time
python - > gpurun_out/r2_nvml_probe.txt 2>&1 <<'PY'
import pynvml as n
n.nvmlInit()
h = n.nvmlDeviceGetHandleByIndex(0)
for fid in (91, 138, 139, 140, 141, 201, 202, 203, 204):
    for scope in (0, 0xffffffff):
        try:
            v = n.nvmlDeviceGetFieldValues(h, [(fid, scope)])[0]
            print(fid, scope, v.nvmlReturn, v.value.ullVal)
        except Exception as e:
            print(fid, scope, "exc", e)
try:
    print("util", n.nvmlDeviceGetNvLinkUtilizationCounter(h, 0, 0))
except Exception as e:
    print("util exc", e)
PY
nvidia-smi nvlink -s -i 0 >> gpurun_out/r2_nvml_probe.txt 2>&1
