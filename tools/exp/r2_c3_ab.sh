# C3 breakdown (ncu launch list) and projector A/B: split-K tile GEMMs vs the fused cluster kernel
set -u
mkdir -p gpurun_out/c3
cd $GRAFT_REPO_ROOT
timeout -s KILL 300 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/c3/launches.csv python tools/prof_c3.py > gpurun_out/c3/prof.log 2>&1; echo "prof rc=$?"
run() {
  timeout -s KILL 600 python bench.py --no-cpu-baseline --no-c4 --no-fit --no-e2e --steps 200 > gpurun_out/c3/$1.json 2> gpurun_out/c3/$1.err
  python -c "
import json; d=json.load(open('gpurun_out/c3/$1.json'))
print('$1', 'value %.0f p50dev %.3f k4proj %.4f sat %s c3 %.0f meshes/s (%.3f ms, lbs %.3f)' % (d['value'], d['frame_latency_device']['p50_ms'], d['stage_ms']['k4_proj_mlp'], d['stage_saturated_us_per_batch'], d['c3']['meshes_per_s'], d['c3']['ms_full'], d['c3']['ms_lbs_fk']))"
}
run split_a
FSB_PROJ_FUSED=1 run fused_a
FSB_PROJ_RESKIN=1 run reskin
run split_b
FSB_PROJ_FUSED=1 run fused_b
