# GPU iteration: parity tests, K3 split, bench (C2 + C3) for FSB_HAND_TPC in $TPCS (default "1")
set -u
mkdir -p gpurun_out/q
timeout -s KILL 900 python -m pytest tests -q -m gpu -x > gpurun_out/q/gputests.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/q/gputests.log
for tpc in ${TPCS:-1}; do
 echo "== FSB_HAND_TPC=$tpc"
 FSB_HAND_TPC=$tpc timeout -s KILL 300 python tools/k3_split.py 2>&1 | tail -5
 FSB_HAND_TPC=$tpc timeout -s KILL 600 python bench.py --no-cpu-baseline --no-c4 --no-fit > gpurun_out/q/bench_tpc$tpc.json 2> gpurun_out/q/bench_tpc$tpc.err; echo "bench rc=$?"
 python -c "
import json; d=json.load(open('gpurun_out/q/bench_tpc$tpc.json'))
print('value %.0f e2e %.0f p50dev %.3f' % (d['value'], d['e2e']['value'] if d.get('e2e') else 0, d['frame_latency_device']['p50_ms']))
print('stages', {k: round(v,4) for k,v in d['stage_ms'].items()}); print('sat', d['stage_saturated_us_per_batch']); r=d['roofline']; print('roof', r['kernel'], r['frac'], r.get('frac_saturated'))
"
done
