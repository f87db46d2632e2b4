cd $GRAFT_REPO_ROOT
python tools/profile_one.py C2 1 > gpurun_out/g21_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_m_cheb -s 44 -c 1 -o gpurun_out/g21_cheb_final python tools/profile_one.py C2 1 > gpurun_out/g21_ncu1.log 2>&1; echo n=$?
python tools/profile_one.py C3 1 > gpurun_out/g21_plain3.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g21_launches_c3.csv python tools/profile_one.py C3 1 > gpurun_out/g21_ncu3.log 2>&1; echo n3=$?
