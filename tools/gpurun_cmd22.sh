cd $GRAFT_REPO_ROOT
{ echo "default"; timeout 120 python tools/percall_probe.py; echo "PS_HOST_DMA=1"; PS_HOST_DMA=1 timeout 120 python tools/percall_probe.py; } > gpurun_out/r2_percall_dma.txt 2>&1
