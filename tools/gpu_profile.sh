#!/bin/bash
# Launch list + one `ncu --set full` capture per hot kernel (run under gpurun,
# one GPU).  Outputs land in gpurun_out/ncu_*.
set -u
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
B="python bench.py --steps 3 --warmup 3 --bank 32 --no-cpu-baseline --no-e2e --no-c3 --no-c4"
timeout -s KILL 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
  --log-file gpurun_out/ncu_launches.csv $B > gpurun_out/ncu_launches.log 2>&1
echo "launch list rc=$?"
for k in k_decoders_tc k_encoder_tc k_boxes_crops k_proj_inputs k_tile_gemm; do
  timeout -s KILL 600 $NCU --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
    -o gpurun_out/ncu_$k -f $B > gpurun_out/ncu_$k.log 2>&1
  echo "ncu $k rc=$?"
done
timeout -s KILL 600 $NCU --set full --clock-control none --import-source on -k regex:k_lbs -s 2 -c 1 \
  -o gpurun_out/ncu_k_lbs_c3 -f python tools/prof_c3.py bf16 > gpurun_out/ncu_k_lbs_c3.log 2>&1
echo "ncu k_lbs c3 rc=$?"
timeout -s KILL 900 $NCU --set full --clock-control none --import-source on -k regex:k_gemm_tc -s 8 -c 4 \
  -o gpurun_out/ncu_c4_gemm -f python tools/prof_c4.py 128 2 > gpurun_out/ncu_c4_gemm.log 2>&1
echo "ncu c4 gemm rc=$?"
timeout -s KILL 600 $NCU --set full --clock-control none --import-source on -k regex:k_attn_tc -s 1 -c 1 \
  -o gpurun_out/ncu_c4_attn -f python tools/prof_c4.py 128 2 > gpurun_out/ncu_c4_attn.log 2>&1
echo "ncu c4 attn rc=$?"
tools/sm_time.sh gpurun_out/sm_time.csv; echo "sm_time rc=$?"
