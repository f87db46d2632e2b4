cd $GRAFT_REPO_ROOT
timeout 300 python bench.py --steps 3 --warmup 3 --config C3 --no-cpu-baseline > gpurun_out/g30_c3.json 2>&1
FMG_LIB=$PWD/paper_2511_19036_b200/libfmg_m3b3.so timeout 300 python bench.py --steps 3 --warmup 3 --config C3 --no-cpu-baseline > gpurun_out/g30_c3_b3.json 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --config C4 --no-cpu-baseline > gpurun_out/g30_c4.json 2>&1
FMG_LIB=$PWD/paper_2511_19036_b200/libfmg_m3b3.so timeout 600 python bench.py --steps 3 --warmup 3 --config C4 --no-cpu-baseline > gpurun_out/g30_c4_b3.json 2>&1
