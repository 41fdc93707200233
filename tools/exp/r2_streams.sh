set -u
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/st
for r in 1 2; do
for S in 12 16 20 24; do
  timeout -s KILL 600 python bench.py --no-cpu-baseline --no-c4 --no-fit --no-e2e --no-c3 --stream-frames 0 --steps 500 --streams $S > gpurun_out/st/$S.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/st/$S.json'))
print('streams $S value %.0f' % d['value'])"
done
done
