cd $GRAFT_REPO_ROOT
t0=$(date +%s); python bench.py > gpurun_out/r2_bench_default.json 2> gpurun_out/r2_bench_default.err; echo "bench_default_wall_s $(( $(date +%s) - t0 ))" >> gpurun_out/r2_bench_default.err
t0=$(date +%s); python bench.py --impl reference > gpurun_out/r2_ref_default.json 2> gpurun_out/r2_ref_default.err; echo "ref_default_wall_s $(( $(date +%s) - t0 ))" >> gpurun_out/r2_ref_default.err
