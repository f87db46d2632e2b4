cd $GRAFT_REPO_ROOT
python tools/profile_one.py C2 1 > gpurun_out/g15_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g15_launches.csv python tools/profile_one.py C2 1 > gpurun_out/g15_ncu0.log 2>&1; echo a=$?
