cd $GRAFT_REPO_ROOT
python tools/profile_one.py C2 1 > gpurun_out/g19_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_m_(residual|cfas1|cheb)" -s 42 -c 3 -o gpurun_out/g19_fine python tools/profile_one.py C2 1 > gpurun_out/g19_ncu.log 2>&1; echo a=$?
