cd $GRAFT_REPO_ROOT
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/g31_base.json 2>&1
for b in 1 2 4 8; do FMG_KC_CLUSTER=1 FMG_KC_BPW=$b FMG_SYNC_DEBUG=1 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/g31_nc1_b$b.json 2> gpurun_out/g31_nc1_b$b.err; done
FMG_KC_CLUSTER=1 FMG_KC_BPW=2 timeout 300 python tools/kc_phases.py C2 > gpurun_out/g31_kc.log 2>&1
