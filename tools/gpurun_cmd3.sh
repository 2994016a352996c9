cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g" 
(time CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_bench_n1.json 2> gpurun_out/r2_bench_n1.err) 2> gpurun_out/r2_bench_n1.time
(time timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r2_bench_n2.json 2> gpurun_out/r2_bench_n2.err) 2> gpurun_out/r2_bench_n2.time
(time timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_ref_n1.json 2> gpurun_out/r2_ref_n1.err) 2> gpurun_out/r2_ref_n1.time
nvidia-smi nvlink -gt d -i 0 > gpurun_out/r2_nvlink_gt.txt 2>&1
