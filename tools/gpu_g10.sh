cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/g10_pytest.log 2>&1; echo pytest=$?
timeout 300 python tools/kc_phases.py C2 > gpurun_out/g10_kc.log 2>&1
FMG_LC=3 timeout 300 python tools/kc_phases.py C2 > gpurun_out/g10_kc3.log 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/g10_bench_c2.json 2>&1; echo b2=$?
FMG_LC=3 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/g10_bench_c2_lc3.json 2>&1; echo b2=$?
