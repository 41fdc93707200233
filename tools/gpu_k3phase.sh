set -u
mkdir -p gpurun_out/k3
python tools/k3_split.py > gpurun_out/k3/k3_split.txt 2>&1; tail -5 gpurun_out/k3/k3_split.txt
FSB_PROFILE=1 python -m paper_2603_15603_b200._build --force > /dev/null 2>&1; echo build rc=$?
python tools/tc_phase_profile.py > gpurun_out/k3/tc_phase.txt 2>&1; cat gpurun_out/k3/tc_phase.txt
