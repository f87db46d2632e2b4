cd $GRAFT_REPO_ROOT
FMG_SYNC_DEBUG=1 timeout 300 python tools/dbg_c3.py 3 1 8,9 > gpurun_out/g3_dbg.log 2>&1
