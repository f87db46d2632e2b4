cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/g17_pytest.log 2>&1; echo pytest=$?
timeout 300 python tools/kc_phases.py C2 > gpurun_out/g17_kc.log 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/g17_bench_c2.json 2>&1; echo b2=$?
for lc in 3 5; do FMG_LC=$lc timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/g17_bench_c2_lc$lc.json 2>&1; done
