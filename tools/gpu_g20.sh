cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv > gpurun_out/g20_smi.csv
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/g20_bench_c2.json 2> gpurun_out/g20_bench_c2.err; echo b2=$?
timeout 600 python bench.py --steps 3 --warmup 3 --config C3 --no-cpu-baseline > gpurun_out/g20_bench_c3.json 2>&1; echo b3=$?
timeout 900 python bench.py --steps 3 --warmup 3 --config C4 --no-cpu-baseline > gpurun_out/g20_bench_c4.json 2>&1; echo b4=$?
timeout 300 python bench.py --steps 3 --warmup 3 --config C1 --no-cpu-baseline > gpurun_out/g20_bench_c1.json 2>&1; echo b1=$?
python tools/profile_one.py C2 1 > gpurun_out/g20_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g20_launches.csv python tools/profile_one.py C2 1 > gpurun_out/g20_ncu0.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_m_cheb -s 62 -c 1 -o gpurun_out/g20_cheb_final python tools/profile_one.py C2 1 > gpurun_out/g20_ncu1.log 2>&1; echo n=$?
