set -u
cd $GRAFT_REPO_ROOT
for v in "2 4" "3 4" "3 8" "2 4" "3 4" "3 8"; do
  set -- $v
  FSB_OBJ_DIR=/tmp/obj_b$1$2 FSB_EXTRA_FLAGS="-DFSB_PROJ_BUFS=$1 -DFSB_PROJ_MPC=$2" python -m paper_2603_15603_b200._build --force > /dev/null 2>&1
  echo "bufs=$1 mpc=$2: $(timeout -s KILL 300 python tools/c3_time.py 2>&1 | tail -1 | cut -c80-170)"
done
