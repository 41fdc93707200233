# A/B: hand tiles per CTA (FSB_HAND_TPC) on the C2 bench, interleaved
set -u
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/tpc
for r in 1 2; do
for v in 0 2; do
  FSB_HAND_TPC=$v timeout -s KILL 600 python bench.py --no-cpu-baseline --no-c4 --no-fit --no-e2e --no-c3 --steps 200 > gpurun_out/tpc/$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/tpc/$v.json'))
print('tpc=$v', 'value %.0f p50dev %.3f k3 %.4f sat %s' % (d['value'], d['frame_latency_device']['p50_ms'], d['stage_ms']['k3_decoders'], d['stage_saturated_us_per_batch']))"
done
done
