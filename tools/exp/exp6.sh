# 384-crop encoder passes: ViT tests (incl. the pass boundary), full GPU suite, C4 twice
mkdir -p gpurun_out/exp6
timeout -s KILL 600 python -m pytest tests -q -m gpu > gpurun_out/exp6/gputests.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/exp6/gputests.log
for i in 1 2; do
  timeout -s KILL 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-c3 --no-fit --no-e2e > gpurun_out/exp6/c4_$i.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/exp6/c4_$i.json'))['c4'];print('c4 ms %.1f tflops %.0f frames/s %.0f'%(d['ms_per_batch'],d['achieved_tflops'],d['frames_per_s']))"
done
