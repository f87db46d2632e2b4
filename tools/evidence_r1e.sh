# Round-1 end-of-session evidence (one gpurun call): GPU tests, smoke, bench
# lines C1-C4 (+ mcgs, nu = 2, the reference arm) and N4, the C2 launch list.
#   /usr/local/graft/bin/gpurun --timeout 2400 -- 'bash tools/evidence_r1e.sh'
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/e_pytest.log 2>&1; echo pytest=$?; tail -1 gpurun_out/e_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/e_smoke.log 2>&1; echo smoke=$?
timeout 600 python bench.py > gpurun_out/e_bench_c2.json 2> gpurun_out/e_bench_c2.err; echo c2=$?
for c in C1 C3 C4; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/e_bench_$c.json 2>/dev/null; echo bench $c $?; done
timeout 300 python bench.py --smoother mcgs --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/e_bench_c2_mcgs.json 2>/dev/null; echo mcgs $?
timeout 300 python bench.py --nu 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/e_bench_c2_nu2.json 2>/dev/null; echo nu2 $?
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/e_bench_c2_reference.json 2>/dev/null; echo ref $?
timeout 300 python bench.py --workload n4 > gpurun_out/e_bench_n4.json 2>/dev/null; echo n4 $?
python tools/profile_one.py C2 1 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/e_c2_launches.csv python tools/profile_one.py C2 1 > /dev/null 2>&1; echo c2list $?
