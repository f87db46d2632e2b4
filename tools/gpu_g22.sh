cd $GRAFT_REPO_ROOT
timeout 300 python tools/kc_phases.py C2 > gpurun_out/g22_kc.log 2>&1
