# LBS occupancy / tiling knobs (FSB_LBS_*): C3 microbench per variant, then C2 for each
mkdir -p gpurun_out/exp4
for n in b200 m16b3g12 m16b4g16 v1b3g6 v1b4g8 m16b2g16 b200; do
  FSB_LIB=$PWD/paper_2603_15603_b200/lib/libfsb_$n.so timeout -s KILL 200 python tools/c3_time.py > gpurun_out/exp4/c3_$n.txt 2>&1
  echo "$n c3: $(tail -1 gpurun_out/exp4/c3_$n.txt | cut -c1-400)"
done
for n in b200 v1b3g6 m16b3g12; do
  FSB_LIB=$PWD/paper_2603_15603_b200/lib/libfsb_$n.so timeout -s KILL 300 python bench.py --no-cpu-baseline --no-c3 --no-c4 --no-fit --no-e2e --steps 2000 > gpurun_out/exp4/c2_$n.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/exp4/c2_$n.json'));print('$n c2 %.0f'%d['value'], d['stage_saturated_us_per_batch'])"
done
