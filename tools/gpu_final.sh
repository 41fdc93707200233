set -u
mkdir -p gpurun_out/final
cd $GRAFT_REPO_ROOT
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/final/smoke.log
timeout -s KILL 900 python -m pytest tests -q -m gpu > gpurun_out/final/gputests.log 2>&1; echo "gpu tests rc=$?"; tail -4 gpurun_out/final/gputests.log
timeout -s KILL 600 python bench.py > gpurun_out/final/bench_bf16.json 2> gpurun_out/final/bench_bf16.err; echo "bench rc=$?"; cut -c1-600 gpurun_out/final/bench_bf16.json
timeout -s KILL 400 python bench.py --impl reference > gpurun_out/final/bench_ref.json 2> gpurun_out/final/bench_ref.err; echo "ref rc=$?"; cut -c1-300 gpurun_out/final/bench_ref.json
timeout -s KILL 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/final/launches.csv python bench.py --steps 3 --warmup 3 --bank 32 --no-cpu-baseline --no-e2e --no-c3 --no-c4 > gpurun_out/final/launches.log 2>&1; echo "launches rc=$?"
timeout -s KILL 600 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:k_decoders_tc -s 2 -c 1 -o gpurun_out/final/ncu_k3 -f python bench.py --steps 3 --warmup 3 --bank 32 --no-cpu-baseline --no-e2e --no-c3 --no-c4 > gpurun_out/final/ncu_k3.log 2>&1; echo "ncu k3 rc=$?"
