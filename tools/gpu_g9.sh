cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/g9_pytest.log 2>&1; echo pytest=$?
timeout 300 python tools/kc_phases.py C2 > gpurun_out/g9_kc.log 2>&1
timeout 300 python tools/timeline.py C2 > gpurun_out/g9_tl.log 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/g9_bench_c2.json 2>&1; echo b2=$?
python tools/profile_one.py C2 1 > gpurun_out/g9_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_op -s 80 -c 3 -o gpurun_out/g9_kop python tools/profile_one.py C2 1 > gpurun_out/g9_ncu.log 2>&1
echo ncu=$?
