set -u
mkdir -p gpurun_out/nc
cd $GRAFT_REPO_ROOT
timeout -s KILL 600 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:"k_lbs_tc|k_proj_inputs_vc" -s 2 -c 2 -o gpurun_out/nc/c3 -f python tools/prof_c3.py > gpurun_out/nc/c3.log 2>&1; echo "ncu rc=$?"
