# C3 launch list + ncu of the bridge kernel + GPU tests
set -u
mkdir -p gpurun_out/it2
cd $GRAFT_REPO_ROOT
timeout -s KILL 900 python -m pytest tests -q -m gpu -x > gpurun_out/it2/gputests.log 2>&1; echo "gpu tests rc=$?"; tail -1 gpurun_out/it2/gputests.log
timeout -s KILL 300 python tools/c3_time.py 2>&1 | tail -1 | cut -c 80-300
timeout -s KILL 300 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/it2/c3_launches.csv python tools/prof_c3.py > gpurun_out/it2/prof.log 2>&1; echo "prof rc=$?"
timeout -s KILL 600 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:"${NCU_K:-k_proj_inputs_vc}" -s 1 -c 1 -o gpurun_out/it2/k -f python tools/prof_c3.py > gpurun_out/it2/ncu.log 2>&1; echo "ncu rc=$?"
