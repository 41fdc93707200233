set -u
cd $GRAFT_REPO_ROOT
for c in 16384 32768 65536; do
  FSB_OBJ_DIR=/tmp/obj_hr FSB_EXTRA_FLAGS="-DFSB_HR_CHUNK=$c" python -m paper_2603_15603_b200._build --force > /dev/null 2>&1
  python -c "
import torch, bench
print('chunk $c', 'sm bulk read %.1f GB/s, copy engine %.1f GB/s' % (bench.host_read_gbs(torch, torch.device('cuda',0)), bench.pinned_h2d_gbs(torch, torch.device('cuda',0))))"
done
