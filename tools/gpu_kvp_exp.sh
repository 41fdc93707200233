set -u
for v in 0 1 2; do
FSB_EXTRA_FLAGS="-DFSB_KVP_EXP=$v" python -m paper_2603_15603_b200._build --force > /dev/null 2>&1; echo "variant $v build rc=$?"
python tools/k3_split.py 2>&1 | grep "encoder+kv"
done
