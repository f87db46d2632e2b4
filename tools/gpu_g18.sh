cd $GRAFT_REPO_ROOT
timeout 300 python tools/timeline.py C2 > gpurun_out/g18_tl.log 2>&1
python tools/profile_one.py C2 1 > gpurun_out/g18_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g18_launches.csv python tools/profile_one.py C2 1 > gpurun_out/g18_ncu0.log 2>&1; echo a=$?
