cd $GRAFT_REPO_ROOT
FMG_SYNC_DEBUG=1 timeout 300 python tools/dbg_c3.py 2 2 3,6 > gpurun_out/g7_dbg.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/g7_pytest.log 2>&1; echo pytest=$?
timeout 300 python tools/kc_phases.py C2 > gpurun_out/g7_kc.log 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/g7_bench_c2.json 2>&1; echo b2=$?
