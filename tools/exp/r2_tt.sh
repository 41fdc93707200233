set -u
cd $GRAFT_REPO_ROOT
timeout -s KILL 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
mkdir -p gpurun_out/tt
for r in 1 2; do
for v in t not; do
  if [ $v = not ]; then export FSB_TILE_NO_T=1; else unset FSB_TILE_NO_T; fi
  timeout -s KILL 600 python bench.py --no-cpu-baseline --no-c4 --no-fit --no-e2e --no-c3 --steps 200 > gpurun_out/tt/$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/tt/$v.json'))
print('$v', 'value %.0f p50dev %.3f k4proj %.4f sat %s' % (d['value'], d['frame_latency_device']['p50_ms'], d['stage_ms']['k4_proj_mlp'], d['stage_saturated_us_per_batch']))"
done
done
