# A/B of the C4 attention kernel (old = libfsb_b200_old.so) + C4 timing, interleaved on one box
set -u
cd $GRAFT_REPO_ROOT
L=paper_2603_15603_b200/lib
timeout -s KILL 600 python -m pytest tests -q -m gpu -x -k "vit or tcgen05" 2>&1 | tail -1
for r in 1 2; do
  for v in old new; do
    if [ $v = old ]; then export FSB_LIB=$PWD/$L/libfsb_b200_old.so; else export FSB_LIB=$PWD/$L/libfsb_b200.so; fi
    echo "$v: $(python tools/attn_time.py 256 576 1024 20 2>&1 | tail -1)"
    echo "$v C4: $(python tools/prof_c4.py 768 24 2>&1 | tail -1 | cut -c150-330)"
  done
done
