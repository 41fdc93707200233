mkdir -p gpurun_out/exp2
for v in b200 fa2; do
  export FSB_LIB=$PWD/paper_2603_15603_b200/lib/libfsb_$v.so
  timeout -s KILL 120 python tools/attn_time.py 256 576 1024 20 >> gpurun_out/exp2/attn.txt 2>&1
  timeout -s KILL 120 python tools/attn_check.py 3 576 1024 >> gpurun_out/exp2/attn.txt 2>&1
  timeout -s KILL 120 python tools/attn_check.py 2 77 128 >> gpurun_out/exp2/attn.txt 2>&1
  timeout -s KILL 300 python -m pytest tests/test_gpu_vit.py -q -x > gpurun_out/exp2/t_vit_$v.txt 2>&1; echo "t_vit $v rc=$?" >> gpurun_out/exp2/attn.txt
  timeout -s KILL 300 python tools/prof_c4.py 768 24 >> gpurun_out/exp2/attn.txt 2>&1
done
cat gpurun_out/exp2/attn.txt
unset FSB_LIB
timeout -s KILL 900 python -m pytest tests -q -m gpu -x > gpurun_out/exp2/gputests.txt 2>&1; echo "gpu tests rc=$?"; tail -n 2 gpurun_out/exp2/gputests.txt
for v in b200 h4 b200 h4; do
  export FSB_LIB=$PWD/paper_2603_15603_b200/lib/libfsb_$v.so
  timeout -s KILL 300 python bench.py --no-cpu-baseline --no-c3 --no-c4 --no-fit --steps 2000 > gpurun_out/exp2/bench_$v.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/exp2/bench_$v.json'));print('$v value %.0f e2e %.0f'%(d['value'],d['e2e']['value']))"
done
