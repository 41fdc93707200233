mkdir -p gpurun_out/exp1
for v in b200 h2 h8 h16; do
  export FSB_LIB=$PWD/paper_2603_15603_b200/lib/libfsb_$v.so
  timeout -s KILL 200 python tools/stage_capacity.py --streams 1,16 > gpurun_out/exp1/cap_$v.txt 2>&1
  timeout -s KILL 300 python bench.py --no-cpu-baseline --no-c3 --no-c4 --no-fit --steps 2000 > gpurun_out/exp1/bench_$v.json 2> gpurun_out/exp1/bench_$v.err
  echo "$v rc=$?"
done
export FSB_LIB=$PWD/paper_2603_15603_b200/lib/libfsb_h8.so
timeout -s KILL 300 python -m pytest tests/test_gpu_bf16.py -q -x > gpurun_out/exp1/t_h8.txt 2>&1; echo "t_h8 rc=$?"
