# on-chip split-K reduction (k_tile_gemm_f) vs partial buffers + k_tile_reduce8 (FSB_TILE_PARTIALS=1)
set -u
mkdir -p gpurun_out/fr
cd $GRAFT_REPO_ROOT
timeout -s KILL 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
run() {
  timeout -s KILL 600 python bench.py --no-cpu-baseline --no-c4 --no-fit --no-e2e --steps 100 $2 > gpurun_out/fr/$1.json 2> gpurun_out/fr/$1.err
  python -c "
import json; d=json.load(open('gpurun_out/fr/$1.json'))
print('$1', 'value %.0f c3 %.0f meshes/s (%.3f ms, lbs %.3f)' % (d['value'], d['c3']['meshes_per_s'], d['c3']['ms_full'], d['c3']['ms_lbs_fk']))"
}
for r in 1 2; do
run fused_$r ""
FSB_TILE_PARTIALS=1 run partials_$r ""
done
run fused_fp32 "--precision fp32"
FSB_TILE_PARTIALS=1 run partials_fp32 "--precision fp32"
