cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 2>&1 | tail -25 > gpurun_out/r2_gpu_all.log
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_bench_n1.json 2> gpurun_out/r2_bench_n1.err
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_ref_n1.json 2> gpurun_out/r2_ref_n1.err
for n in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2962$n bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/r2_bench_n$n.json 2> gpurun_out/r2_bench_n$n.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2963$n bench.py --impl reference --gpus $n --steps 20 --warmup 5 > gpurun_out/r2_ref_n$n.json 2> gpurun_out/r2_ref_n$n.err
done
CUDA_VISIBLE_DEVICES=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches_n1.csv python bench.py --steps 3 --warmup 3 --no-sweep > gpurun_out/r2_ncu_launch.log 2>&1
