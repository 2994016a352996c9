cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_replay.py tests/test_gpu_freerun.py tests/test_gpu_gate.py -q -x 2>&1 | tail -3 > gpurun_out/r2_t40.log
{ for sc in 0 1; do for p in dssp ssp bsp asp; do for m in full gate data; do PS_REPLAY_GATE_SCAN=$sc timeout 120 python tools/replay_paradigm.py $p $m | sed "s/^/scan=$sc /"; done; done; done; } > gpurun_out/r2_scan.txt 2>&1
{ for c in 18 37 74; do echo "ctas=$c"; PS_WORKERS_CTAS=$c timeout 120 python tools/nvlink_probe.py 16777216 40; PS_WORKERS_CTAS=$c timeout 120 python tools/nvlink_probe.py 1730714 100; done; echo default; timeout 120 python tools/nvlink_probe.py 16777216 40; timeout 120 python tools/nvlink_probe.py 1730714 100; } > gpurun_out/r2_wctas2.txt 2>&1
timeout 300 python bench.py --steps 20 --warmup 3 > gpurun_out/r2_b40.json 2> gpurun_out/r2_b40.err
