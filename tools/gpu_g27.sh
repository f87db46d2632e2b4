cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/g27_pytest.log 2>&1; echo pytest=$?
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/g27_bench.json 2>&1; echo b2=$?
python tools/profile_one.py C2 1 > gpurun_out/g27_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g27_launches.csv python tools/profile_one.py C2 1 > gpurun_out/g27_ncu0.log 2>&1; echo n=$?
