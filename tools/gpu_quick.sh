# quick GPU iteration: parity tests (-x), K3 split timing, optional bench
set -u
mkdir -p gpurun_out/q
timeout -s KILL 900 python -m pytest tests -q -m gpu -x ${PYTEST_ARGS:-} > gpurun_out/q/gputests.log 2>&1; echo "gpu tests rc=$?"; tail -15 gpurun_out/q/gputests.log
timeout -s KILL 300 python tools/k3_split.py > gpurun_out/q/k3_split.txt 2>&1; tail -4 gpurun_out/q/k3_split.txt
if [ -n "${BENCH:-}" ]; then
  timeout -s KILL 600 python bench.py --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/q/bench.json 2> gpurun_out/q/bench.err; echo "bench rc=$?"
  python -c "
import json; d=json.load(open('gpurun_out/q/bench.json'))
print('value %.0f e2e %.0f p50dev %.3f' % (d['value'], d['e2e']['value'] if d.get('e2e') else 0, d['frame_latency_device']['p50_ms']))
print('stages', d['stage_ms']); print('sat', d['stage_saturated_us_per_batch']); r=d['roofline']; print('roof', r['kernel'], r['frac'], r.get('frac_saturated'))
"
fi
