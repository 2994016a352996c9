set -x
timeout 300 python -m pytest tests/test_gpu_sharded.py -x -q 2>&1 | tail -5
for w in 2 4; do
timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node $w --master-addr 127.0.0.1 --master-port 2950$w tools/shard_probe.py 4096 2>&1 | grep world
timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node $w --master-addr 127.0.0.1 --master-port 2951$w tools/shard_probe.py 2>&1 | grep world
done
timeout 120 ./tools/p2p_alltoall 2>&1 | tail -20
