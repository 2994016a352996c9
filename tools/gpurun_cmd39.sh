cd $GRAFT_REPO_ROOT
timeout 800 python -m pytest tests/test_gpu_freerun.py -q 2>&1 | tail -3 > gpurun_out/r2_t39.log
{ for c in 18 37 74; do echo "ctas=$c"; PS_WORKERS_CTAS=$c timeout 120 python tools/nvlink_probe.py 16777216 10; PS_WORKERS_CTAS=$c timeout 120 python tools/nvlink_probe.py 1730714 20; done; echo default; timeout 120 python tools/nvlink_probe.py 16777216 10; } > gpurun_out/r2_wctas.txt 2>&1
timeout 600 python -c "
import sys, json, torch
sys.argv=['bench.py']
import bench
import paper_1908_11848_b200 as ps
out = bench.free_running(torch, ps, 110, 3, (1.0,2.0,4.0), 24)
print(json.dumps(out))
out = bench.free_running(torch, ps, 110, 3, (1.0,2.0,4.0), 24, devices=[0,1,0])
print(json.dumps(out))
" > gpurun_out/r2_fr3.json 2> gpurun_out/r2_fr3.err
