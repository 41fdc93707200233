# LBS variants at C3: joint stride (FSB_LBS_JS) x corner write scheme (FSB_LBS_URUN)
set -u
mkdir -p gpurun_out/lv
cd $GRAFT_REPO_ROOT
for v in "14 1" "14 0" "12 0" "12 1" "16 1"; do
  set -- $v
  FSB_EXTRA_FLAGS="-DFSB_LBS_JS=$1 -DFSB_LBS_URUN=$2" python -m paper_2603_15603_b200._build --force > /dev/null 2>&1
  echo "JS=$1 URUN=$2: $(timeout -s KILL 300 python tools/c3_time.py 2>&1 | tail -1 | cut -c1-400)"
done
python -m paper_2603_15603_b200._build --force > /dev/null 2>&1
timeout -s KILL 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum --clock-control none -k regex:"k_lbs_tc|k_proj_inputs" --csv --log-file gpurun_out/lv/launches.csv python tools/prof_c3.py > gpurun_out/lv/prof.log 2>&1; echo "prof rc=$?"
