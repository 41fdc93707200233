set -u
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/lbsg
for r in 1 2; do
for v in 1 2 4; do
  FSB_LBS_MINCH=$v timeout -s KILL 600 python bench.py --no-cpu-baseline --no-c4 --no-fit --no-e2e --steps 200 > gpurun_out/lbsg/$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/lbsg/$v.json'))
print('minch=$v', 'value %.0f p50dev %.3f sat %s c3 %.3f' % (d['value'], d['frame_latency_device']['p50_ms'], d['stage_saturated_us_per_batch'], d['c3']['ms_full']))"
done
done
