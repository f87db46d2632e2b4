# Round-2 evidence, final build of the second session (one gpurun call): bench lines, launch lists and the ncu
# capture of the roofline kernel.  /usr/local/graft/bin/gpurun --timeout 3000 -- 'bash tools/evidence_r2c.sh'
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ev3
make -s -C oracle > /dev/null 2>&1
nproc > gpurun_out/ev3/nproc.txt
B="timeout 900 python bench.py"
$B > gpurun_out/ev3/bench_C4.json 2> gpurun_out/ev3/bench_C4.err; echo C4 $?
for c in C3 C2 C1 C5h; do $B --config $c --steps 5 --warmup 3 > gpurun_out/ev3/bench_$c.json 2> gpurun_out/ev3/bench_$c.err; echo $c $?; done
$B --cfas-fp32 --steps 5 --warmup 3 > gpurun_out/ev3/bench_C4_fp32.json 2>/dev/null; echo C4fp32 $?
$B --config C3 --cfas-fp32 --steps 5 --warmup 3 > gpurun_out/ev3/bench_C3_fp32.json 2>/dev/null; echo C3fp32 $?
FMG_F3MAT=0 $B --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ev3/bench_C4_lean.json 2>/dev/null; echo C4lean $?
$B --impl reference --steps 3 --warmup 3 > gpurun_out/ev3/bench_C4_reference.json 2>/dev/null; echo ref $?
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/ev3/pytest.log 2>&1; echo pytest $?
timeout 300 python tools/profile_one.py C4 1 > /dev/null 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/ev3/c4_launches.csv python tools/profile_one.py C4 1 > /dev/null 2>&1; echo list4 $?
timeout 300 python tools/profile_one.py C4 1 fp32 > /dev/null 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/ev3/c4_fp32_launches.csv python tools/profile_one.py C4 1 fp32 > /dev/null 2>&1; echo list4f $?
timeout 300 python tools/profile_one.py C3 1 > /dev/null 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/ev3/c3_launches.csv python tools/profile_one.py C3 1 > /dev/null 2>&1; echo list3 $?
RX="k_f3|k_m3_restrict"
SK=$(python tools/launches.py --skip gpurun_out/ev3/c4_launches.csv "$RX" k_f3_prolong 8); echo skip $SK
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$RX" -s $SK -c 8 -o gpurun_out/ev3/c4_full python tools/profile_one.py C4 1 > gpurun_out/ev3/ncu_full.log 2>&1; echo full $?
