# round-2 iteration: GPU tests + short bench (no CPU arm / e2e / C4 / fit)
set -u
mkdir -p gpurun_out/it
cd $GRAFT_REPO_ROOT
timeout -s KILL 900 python -m pytest tests -q -m gpu -x > gpurun_out/it/gputests.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/it/gputests.log
timeout -s KILL 600 python bench.py --no-cpu-baseline --no-c4 --no-fit --no-e2e --steps 200 > gpurun_out/it/bench.json 2> gpurun_out/it/bench.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/it/bench.json'))
print('value %.0f p50dev %.3f sat %s c3 %.0f meshes/s (%.3f ms, lbs %.3f)' % (d['value'], d['frame_latency_device']['p50_ms'], d['stage_saturated_us_per_batch'], d['c3']['meshes_per_s'], d['c3']['ms_full'], d['c3']['ms_lbs_fk']))"
if [ -n "${NCU_C3:-}" ]; then
timeout -s KILL 300 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/it/c3_launches.csv python tools/prof_c3.py > gpurun_out/it/prof.log 2>&1; echo "prof rc=$?"
fi
