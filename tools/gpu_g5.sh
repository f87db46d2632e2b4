cd $GRAFT_REPO_ROOT
timeout 300 python tools/kc_phases.py C2 > gpurun_out/g5_kc.log 2>&1
timeout 300 python tools/timeline.py C2 > gpurun_out/g5_tl_c2.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/g5_pytest.log 2>&1; echo pytest=$?
