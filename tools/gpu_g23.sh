cd $GRAFT_REPO_ROOT
for b in 1 2 4; do FMG_KC_BPW=$b FMG_SYNC_DEBUG=1 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/g23_bench_bpw$b.json 2> gpurun_out/g23_bpw$b.err; done
FMG_KC_BPW=2 timeout 300 python tools/kc_phases.py C2 > gpurun_out/g23_kc.log 2>&1
