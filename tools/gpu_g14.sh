cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/g14_pytest.log 2>&1; echo pytest=$?
