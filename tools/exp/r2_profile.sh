#!/bin/bash
# Round-2 evidence: launch list + one `ncu --set full` capture per hot kernel
# (C2 stages on one 32-frame batch, C3 kernels at 4096 meshes, C4 GEMM and
# attention) + SM-time of one batch.  Outputs in gpurun_out/r2p/.
set -u
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2p
mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
B="python bench.py --steps 3 --warmup 3 --bank 32 --no-cpu-baseline --no-e2e --no-c3 --no-c4 --no-fit --stream-frames 0"
timeout -s KILL 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file $O/launches.csv $B > $O/launches.log 2>&1
echo "launch list rc=$?"
S="python tools/prof_stages.py --precision bf16"
for k in k_decoders_tc k_encoder_tc k_boxes_crops k_lbs_tc k_proj_inputs_vc k_tile_gemm; do
  timeout -s KILL 600 $NCU --set full --clock-control none --import-source on -k regex:"^$k" -s 2 -c 1 -o $O/c2_$k -f $S > $O/c2_$k.log 2>&1
  echo "ncu c2 $k rc=$?"
done
for k in k_lbs_tc k_proj_inputs_vc k_tile_gemm_p; do
  timeout -s KILL 600 $NCU --set full --clock-control none --import-source on -k regex:"^$k" -s 0 -c 1 -o $O/c3_$k -f python tools/prof_c3.py bf16 > $O/c3_$k.log 2>&1
  echo "ncu c3 $k rc=$?"
done
timeout -s KILL 900 $NCU --set full --clock-control none --import-source on -k regex:k_gemm_tc -s 8 -c 4 -o $O/c4_gemm -f python tools/prof_c4.py 256 2 > $O/c4_gemm.log 2>&1
echo "ncu c4 gemm rc=$?"
timeout -s KILL 600 $NCU --set full --clock-control none --import-source on -k regex:k_attn_tc -s 1 -c 1 -o $O/c4_attn -f python tools/prof_c4.py 256 2 > $O/c4_attn.log 2>&1
echo "ncu c4 attn rc=$?"
bash tools/sm_time.sh $O/sm_time.csv > $O/sm_time.log 2>&1; echo "sm_time rc=$?"
