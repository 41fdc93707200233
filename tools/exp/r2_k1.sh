set -u
cd $GRAFT_REPO_ROOT
L=$PWD/paper_2603_15603_b200/lib
timeout -s KILL 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -1
mkdir -p gpurun_out/k1
for r in 1 2; do
for v in new old; do
  if [ $v = old ]; then export FSB_LIB=$L/libfsb_b200_old.so; else export FSB_LIB=$L/libfsb_b200.so; fi
  timeout -s KILL 600 python bench.py --no-cpu-baseline --no-c4 --no-fit --no-e2e --no-c3 --steps 200 > gpurun_out/k1/$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/k1/$v.json'))
print('$v', 'value %.0f k1 %.4f sat %s' % (d['value'], d['stage_ms']['k1_boxes_crops'], d['stage_saturated_us_per_batch']))"
done
done
