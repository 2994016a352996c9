cd $GRAFT_REPO_ROOT
bash tools/gpurun_cmd56.sh
bash tools/gpurun_cmd62.sh
