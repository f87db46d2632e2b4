# Round-1 final evidence (one gpurun call): GPU tests, bench lines C1-C4 + mcgs,
# C2/C3 launch lists.   /usr/local/graft/bin/gpurun --timeout 2400 -- 'bash tools/evidence_r1d.sh'
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/d_pytest.log 2>&1; echo pytest=$?
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/d_bench_c2.json 2> gpurun_out/d_bench_c2.err; echo c2=$?
for c in C1 C3 C4; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/d_bench_$c.json 2>/dev/null; echo bench $c $?; done
timeout 300 python bench.py --smoother mcgs --steps 10 --warmup 3 > gpurun_out/d_bench_c2_mcgs.json 2>/dev/null; echo mcgs $?
python tools/profile_one.py C2 1 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/d_c2_launches.csv python tools/profile_one.py C2 1 > /dev/null 2>&1; echo c2list $?
python tools/profile_one.py C3 1 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/d_c3_launches.csv python tools/profile_one.py C3 1 > /dev/null 2>&1; echo c3list $?
