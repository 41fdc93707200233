# C3 / C2 A/B of libfsb_b200_old.so vs libfsb_b200.so (GPU tests on new first)
set -u
mkdir -p gpurun_out/c3ab
cd $GRAFT_REPO_ROOT
L=$PWD/paper_2603_15603_b200/lib
timeout -s KILL 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -1
for r in 1 2; do
for v in new old; do
  if [ $v = old ]; then export FSB_LIB=$L/libfsb_b200_old.so; else export FSB_LIB=$L/libfsb_b200.so; fi
  timeout -s KILL 600 python bench.py --no-cpu-baseline --no-c4 --no-fit --no-e2e --steps 100 > gpurun_out/c3ab/$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/c3ab/$v.json'))
print('$v', 'value %.0f p50dev %.3f proj %.2f c3 %.0f meshes/s (%.3f ms, lbs %.3f)' % (d['value'], d['frame_latency_device']['p50_ms'], d['stage_saturated_us_per_batch']['k4_proj_mlp'], d['c3']['meshes_per_s'], d['c3']['ms_full'], d['c3']['ms_lbs_fk']))"
done
done
