# generic A/B of libfsb_b200_old.so vs libfsb_b200.so: GPU tests on new, K3 split + C2 bench interleaved
set -u
cd $GRAFT_REPO_ROOT
L=$PWD/paper_2603_15603_b200/lib
timeout -s KILL 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -1
mkdir -p gpurun_out/ab
for r in 1 2; do
for v in new old; do
  if [ $v = old ]; then export FSB_LIB=$L/libfsb_b200_old.so; else export FSB_LIB=$L/libfsb_b200.so; fi
  echo "$v k3: $(python tools/k3_split.py 2>&1 | tail -5 | tr '\n' ' ')"
  timeout -s KILL 600 python bench.py --no-cpu-baseline --no-c4 --no-fit --no-e2e --no-c3 --steps 200 > gpurun_out/ab/$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ab/$v.json'))
print('$v', 'value %.0f p50dev %.3f sat %s' % (d['value'], d['frame_latency_device']['p50_ms'], d['stage_saturated_us_per_batch']))"
done
done
