set -u
cd $GRAFT_REPO_ROOT
for w in 8 16 8 16; do
  FSB_OBJ_DIR=/tmp/obj_w$w FSB_EXTRA_FLAGS="-DFSB_LBS_WARPS=$w" python -m paper_2603_15603_b200._build --force > /dev/null 2>&1
  echo "warps=$w: $(timeout -s KILL 300 python tools/c3_time.py 2>&1 | tail -1 | cut -c80-210)"
done
