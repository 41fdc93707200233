# LBS tile grouping A/B: cost-balanced 64-vertex blocks per tile vs consecutive blocks (FSB_LBS_NATURAL=1)
set -u
mkdir -p gpurun_out/lbsbal
cd $GRAFT_REPO_ROOT
timeout -s KILL 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -1
run() {
  timeout -s KILL 600 python bench.py --no-cpu-baseline --no-c4 --no-fit --no-e2e --steps 200 > gpurun_out/lbsbal/$1.json 2> gpurun_out/lbsbal/$1.err
  python -c "
import json; d=json.load(open('gpurun_out/lbsbal/$1.json'))
print('$1', 'value %.0f sat %s c3 %.0f meshes/s (%.3f ms, lbs %.3f)' % (d['value'], d['stage_saturated_us_per_batch'], d['c3']['meshes_per_s'], d['c3']['ms_full'], d['c3']['ms_lbs_fk']))"
}
for r in 1 2; do
run bal_$r
FSB_LBS_NATURAL=1 run nat_$r
done
