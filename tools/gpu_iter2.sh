# GPU iteration: parity tests (-x), K3 split timing, FSB_PROFILE phase split
set -u
mkdir -p gpurun_out/q
timeout -s KILL 900 python -m pytest tests -q -m gpu -x ${PYTEST_ARGS:-} > gpurun_out/q/gputests.log 2>&1; echo "gpu tests rc=$?"; tail -4 gpurun_out/q/gputests.log
bash tools/gpu_k3phase.sh
