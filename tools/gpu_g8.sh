cd $GRAFT_REPO_ROOT
python tools/profile_one.py C2 2 > gpurun_out/g8_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:kc_kernel -s 6 -c 1 -o gpurun_out/g8_kc python tools/profile_one.py C2 2 > gpurun_out/g8_ncu.log 2>&1
echo ncu=$?
