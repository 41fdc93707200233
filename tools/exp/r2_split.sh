set -u
cd $GRAFT_REPO_ROOT
timeout -s KILL 900 python -m pytest tests -q -m gpu 2>&1 | tail -4
mkdir -p gpurun_out/split
for v in split simt; do
  if [ $v = simt ]; then export FSB_MLP_SIMT=1; else unset FSB_MLP_SIMT; fi
  timeout -s KILL 600 python bench.py --precision fp32 --no-cpu-baseline --no-c4 --no-fit --no-e2e --steps 100 > gpurun_out/split/$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/split/$v.json'))
print('$v', 'value %.0f p50dev %.3f sat %s c3 %.3f ms' % (d['value'], d['frame_latency_device']['p50_ms'], d['stage_saturated_us_per_batch'], d['c3']['ms_full']))"
done
