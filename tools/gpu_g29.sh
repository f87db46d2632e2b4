cd $GRAFT_REPO_ROOT
nproc > gpurun_out/g29_nproc.txt; free -g >> gpurun_out/g29_nproc.txt
timeout 300 python bench.py --steps 5 --warmup 3 --smoother mcgs > gpurun_out/g29_bench_c2_mcgs.json 2>&1; echo b=$?
timeout 300 python bench.py --steps 3 --warmup 3 --smoother mcgs --config C3 --no-cpu-baseline > gpurun_out/g29_bench_c3_mcgs.json 2>&1; echo b=$?
FMG_FULL_ORACLE=1 timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k C3_full_oracle > gpurun_out/g29_c3_oracle.log 2>&1; echo t=$?
