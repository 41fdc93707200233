# same-box A/B of the encoder pass size: 384 (default) vs 256, interleaved
mkdir -p gpurun_out/exp7
for n in b200 vc256 b200 vc256 b200 vc256; do
  FSB_LIB=$PWD/paper_2603_15603_b200/lib/libfsb_$n.so timeout -s KILL 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-c3 --no-fit --no-e2e > gpurun_out/exp7/$n.json 2>/dev/null
  python -c "import json;D=json.load(open('gpurun_out/exp7/$n.json'));d=D['c4'];print('$n c4 ms %.1f tflops %.0f'%(d['ms_per_batch'],d['achieved_tflops']), D['clocks'])"
done
