cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/g12_pytest.log 2>&1; echo pytest=$?
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --config C3 > gpurun_out/g12_bench_c3.json 2>&1; echo b3=$?
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --config C4 > gpurun_out/g12_bench_c4.json 2>&1; echo b4=$?
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/g12_bench_c2.json 2>&1; echo b2=$?
timeout 300 python tools/timeline.py C3 > gpurun_out/g12_tl_c3.log 2>&1
