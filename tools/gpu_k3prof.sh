set -u
mkdir -p gpurun_out
python -m pytest tests/test_gpu_r2.py -q -s -k "vitl_24 or render_scene" -p no:cacheprovider 2>&1 | grep -E "rel-L2|fraction|passed|failed" 
python tools/k3_split.py > gpurun_out/k3_split.txt 2>&1; cat gpurun_out/k3_split.txt | tail -5
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_decoders_tc -s 2 -c 1 -o gpurun_out/ncu_k3_r2 -f python tools/prof_stages.py --precision bf16 > gpurun_out/ncu_k3.log 2>&1; echo ncu rc=$?
FSB_PROFILE=1 python -m paper_2603_15603_b200._build --force > /dev/null 2>&1; echo build rc=$?
python tools/tc_phase_profile.py > gpurun_out/tc_phase.txt 2>&1; cat gpurun_out/tc_phase.txt
