# One gpurun call: GPU parity tests, the default bench line, and the ncu launch
# list of one C2 solve (profiles/ summaries are derived from these).
#   /usr/local/graft/bin/gpurun --timeout 1800 -- 'bash tools/gpu_check.sh'
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/check_pytest.log 2>&1; echo pytest=$?
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/check_bench.json 2> gpurun_out/check_bench.err; echo bench=$?
python tools/profile_one.py C2 1 > gpurun_out/check_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/check_launches.csv \
    python tools/profile_one.py C2 1 > gpurun_out/check_ncu.log 2>&1; echo ncu=$?
