# C4 crops per encoder pass (FSB_VIT_CHUNK): 128 / 256 (default) / 384 / 768
mkdir -p gpurun_out/exp5
for n in b200 vc128 vc384 vc768 b200; do
  FSB_LIB=$PWD/paper_2603_15603_b200/lib/libfsb_$n.so timeout -s KILL 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-c3 --no-fit --no-e2e > gpurun_out/exp5/$n.json 2>gpurun_out/exp5/$n.err
  python -c "import json;d=json.load(open('gpurun_out/exp5/$n.json'))['c4'];print('$n c4 ms %.1f tflops %.0f'%(d['ms_per_batch'],d['achieved_tflops']))"
done
