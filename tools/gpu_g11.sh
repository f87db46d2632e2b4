cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/g11_pytest.log 2>&1; echo pytest=$?
timeout 300 python tools/timeline.py C2 > gpurun_out/g11_tl.log 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/g11_bench_c2.json 2>&1; echo b2=$?
FMG_MARCH=0 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/g11_bench_c2_nomarch.json 2>&1; echo b2=$?
