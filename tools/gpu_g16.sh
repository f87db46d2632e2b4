cd $GRAFT_REPO_ROOT
python tools/profile_one.py C2 1 > gpurun_out/g16_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:kc_kernel -s 0 -c 2 -o gpurun_out/g16_kc python tools/profile_one.py C2 1 > gpurun_out/g16_ncu.log 2>&1; echo a=$?
