set -u
mkdir -p gpurun_out/c4
cd $GRAFT_REPO_ROOT
timeout -s KILL 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/c4/launches.csv python tools/prof_c4.py 768 2 > gpurun_out/c4/prof.log 2>&1; echo "prof rc=$?"
