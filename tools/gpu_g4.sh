cd $GRAFT_REPO_ROOT
FMG_SYNC_DEBUG=1 timeout 300 python tools/dbg_c3.py 2 1 3,5 > gpurun_out/g4_dbg.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/g4_pytest.log 2>&1; echo pytest=$?
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/g4_bench_c2.json 2>&1; echo b2=$?
timeout 300 python tools/timeline.py C2 > gpurun_out/g4_tl_c2.log 2>&1
