cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
( timeout 900 compute-sanitizer --tool memcheck --leak-check no --print-limit 20 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_freerun.py -k "synthetic and dssp and True" 2>&1 | tail -15 ) > gpurun_out/r2_sanitizer_freerun.log
( timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_server.py -k "bit_exact or device_tensor or divergence or rejected or retires" 2>&1 | tail -15 ) > gpurun_out/r2_sanitizer_server.log
( timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/shard_one.py 4099 2>&1 | tail -8 ) > gpurun_out/r2_sanitizer_shard.log
( timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python tools/replay_paradigm.py dssp full 2>&1 | tail -8 ) > gpurun_out/r2_racecheck_replay.log
timeout 300 python tools/apply_sweep_probe.py > gpurun_out/r2_apply_small3.txt 2>&1
