cd $GRAFT_REPO_ROOT
FMG_SYNC_DEBUG=1 timeout 300 python tools/dbg_c3.py 2 2 7 > gpurun_out/g26_dbg.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/g26_pytest.log 2>&1; echo pytest=$?
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/g26_bench.json 2>&1; echo b2=$?
FMG_PIPE=0 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/g26_bench_nopipe.json 2>&1; echo b2=$?
