set -u
mkdir -p gpurun_out/k3
for v in 1 2; do
FSB_PROFILE=1 FSB_EXTRA_FLAGS="-DFSB_HKV_EXP=$v" python -m paper_2603_15603_b200._build --force > /dev/null 2>&1; echo "variant $v build rc=$?"
python tools/tc_phase_profile.py 2>&1 | grep -A1 "hand decoder t0" | head -2
done
