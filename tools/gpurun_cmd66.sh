cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_freerun.py -q -x 2>&1 | tail -5 > gpurun_out/r2_t66.log
timeout 600 python -c "
import sys, json, torch
sys.argv=['bench.py']
import bench
import paper_1908_11848_b200 as ps
out = bench.free_running(torch, ps, 110, 3, (1.0,2.0,4.0), 24, devices=[0,1,2])
print(json.dumps(out))
" > gpurun_out/r2_fr4.json 2> gpurun_out/r2_fr4.err
