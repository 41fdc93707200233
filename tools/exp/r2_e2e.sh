set -u
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/e2e
for v in 6 10 16 6 10 16; do
  FSB_E2E_STREAMS=$v timeout -s KILL 600 python bench.py --no-cpu-baseline --no-c4 --no-fit --no-c3 --stream-frames 0 --steps 40 > gpurun_out/e2e/$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/e2e/$v.json'))
e=d['e2e']; print('streams=$v e2e %.0f frames/s  %.1f GB/s  frac %.3f peak %.1f (copy %.1f, sm %.1f)' % (e['value'], e['roofline']['achieved'], e['roofline']['frac'], e['roofline']['peak'], e['roofline']['peak_copy_engine_gbs'], e['roofline']['peak_sm_bulk_read_gbs']))"
done
