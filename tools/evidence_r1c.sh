cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
bash tools/gpu_check.sh
for c in C1 C3 C4; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/ev_bench_$c.json 2>/dev/null; echo bench $c $?; done
timeout 300 python bench.py --smoother mcgs --steps 10 --warmup 3 > gpurun_out/ev_bench_c2_mcgs.json 2>/dev/null; echo mcgs $?
python tools/profile_one.py C3 1 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev_c3_launches.csv python tools/profile_one.py C3 1 > /dev/null 2>&1; echo c3list $?
ncu --set full --import-source on --clock-control none -k regex:k_m3_cheb --launch-skip 44 --launch-count 1 -o gpurun_out/ev_c3_cheb python tools/profile_one.py C3 1 > gpurun_out/ev_ncu.log 2>&1; echo ncu $?
