set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/g1_pytest.log 2>&1; echo pytest=$?
timeout 300 python bench.py --steps 5 --warmup 3 > gpurun_out/g1_bench_c2.json 2> gpurun_out/g1_bench_c2.err; echo b2=$?
timeout 300 python bench.py --steps 3 --warmup 3 --config C1 --no-cpu-baseline > gpurun_out/g1_bench_c1.json 2>&1; echo b1=$?
timeout 600 python bench.py --steps 3 --warmup 3 --config C3 --no-cpu-baseline > gpurun_out/g1_bench_c3.json 2>&1; echo b3=$?
timeout 600 python bench.py --steps 3 --warmup 3 --config C4 --no-cpu-baseline > gpurun_out/g1_bench_c4.json 2>&1; echo b4=$?
