cd $GRAFT_REPO_ROOT
mkdir -p /tmp/sv
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29610 tests/_sharded_worker.py /tmp/sv > gpurun_out/r2_sv.log 2>&1
cat /tmp/sv/rank0.json >> gpurun_out/r2_sv.log 2>/dev/null
timeout 900 python -m pytest tests/test_gpu_acceptance.py -q -x 2>&1 | tail -15 > gpurun_out/r2_acc.log
for u in 1 2 4; do PS_APPLY_SMALL_U=$u timeout 300 python tools/apply_sweep_probe.py; done > gpurun_out/r2_apply_small.txt 2>&1
timeout 120 python tools/percall_probe.py > gpurun_out/r2_percall.txt 2>&1
