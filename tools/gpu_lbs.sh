set -u
python tools/lbs_repro.py 32 2>&1 | tail -1
python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "skin or c3 or lbs or frame or smoke or perturbed or toy or oof" 2>&1 | tail -2
for i in 1 2; do
  python tools/c3_time.py 2>&1 | tail -1 | cut -c 100-260
done
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:k_lbs_tc -s 2 -c 1 -o gpurun_out/ncu_lbs_tc -f python tools/prof_c3.py bf16 > gpurun_out/ncu_lbs_tc.log 2>&1; echo ncu rc=$?
