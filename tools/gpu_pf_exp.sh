# A/B: projector unfused vs fused cluster kernel (CS 16 / 8)
set -u
mkdir -p gpurun_out/pf
run() {
  timeout -s KILL 600 python bench.py --no-cpu-baseline --no-c4 --no-fit --no-e2e > gpurun_out/pf/$1.json 2> gpurun_out/pf/$1.err
  python -c "
import json; d=json.load(open('gpurun_out/pf/$1.json'))
print('$1', 'value %.0f p50dev %.3f k4proj %.4f sat %.2f c3 %.0f meshes/s (%.3f ms)' % (d['value'], d['frame_latency_device']['p50_ms'], d['stage_ms']['k4_proj_mlp'], d['stage_saturated_us_per_batch']['k4_proj_mlp'], d['c3']['meshes_per_s'], d['c3']['ms_full']))"
}
FSB_PROJ_UNFUSED=1 run unfused
run fused16
FSB_EXTRA_FLAGS="-DFSB_PF_CS=8" python -m paper_2603_15603_b200._build --force > /dev/null 2>&1
run fused8
FSB_PROJ_UNFUSED=1 run unfused_b
