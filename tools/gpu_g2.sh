cd $GRAFT_REPO_ROOT
timeout 300 python tools/dbg_c3.py 3 1 6,7,8,9 > gpurun_out/g2_dbg.log 2>&1
CUDA_LAUNCH_BLOCKING=1 timeout 300 python tools/dbg_c3.py 3 1 9 > gpurun_out/g2_dbg_blk.log 2>&1
timeout 300 python tools/timeline.py C4 > gpurun_out/g2_tl_c4.log 2>&1
timeout 300 python tools/timeline.py C2 > gpurun_out/g2_tl_c2.log 2>&1
