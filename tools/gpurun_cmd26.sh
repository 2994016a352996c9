cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke2.log 2>&1
{ for cps in 1 2; do for lib in paper_1908_11848_b200/libdssp_ps.so tools/libdssp_ps_M2.so; do echo "cps=$cps lib=$lib"; PS_SIM_CTAS_PER_SM=$cps DSSP_PS_LIB=$lib timeout 120 python tools/replay_paradigm.py dssp data; PS_SIM_CTAS_PER_SM=$cps DSSP_PS_LIB=$lib timeout 120 python tools/replay_paradigm.py dssp full; done; done; } > gpurun_out/r2_sim_occupancy.txt 2>&1
