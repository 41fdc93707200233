# hands-per-tile 6 / 12 and the in-flight stream count with the 8-hand default
mkdir -p gpurun_out/exp3
run() {  # name lib streams
  FSB_LIB=$PWD/paper_2603_15603_b200/lib/libfsb_$2.so timeout -s KILL 300 python bench.py --no-cpu-baseline --no-c3 --no-c4 --no-fit --no-e2e --steps 2000 --streams $3 > gpurun_out/exp3/bench_$1.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/exp3/bench_$1.json'));print('$1 value %.0f'%d['value'])"
}
run h6 h6 16; run h12 h12 16; run s16 b200 16
for s in 12 20 24 32; do run s$s b200 $s; done
run s16b b200 16; run h12b h12 16
