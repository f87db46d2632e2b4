cd $GRAFT_REPO_ROOT
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/g25_base.json 2>&1
FMG_LIB=$PWD/paper_2511_19036_b200/libfmg_minb4.so timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/g25_minb4.json 2>&1
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --config C3 > gpurun_out/g25_base_c3.json 2>&1
FMG_LIB=$PWD/paper_2511_19036_b200/libfmg_minb4.so timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --config C3 > gpurun_out/g25_minb4_c3.json 2>&1
