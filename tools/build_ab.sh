# Build libtn.so of git revision $1 (default HEAD) into build_ab/libtn_B.so for a same-box A/B
# (tools/gpu_ab.sh with AB_ENV_B="TN_LIB_PATH=$PWD/build_ab/libtn_B.so"; the .so travels with gpurun).
set -e
REV=${1:-HEAD}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
W=/tmp/tn_ab_worktree
rm -rf $W; git -C $ROOT worktree prune
git -C $ROOT worktree add -f $W $REV > /dev/null
(cd $W && python -c "from paper_2310_03978_b200 import _build; _build.build(force=True)")
mkdir -p $ROOT/build_ab
cp $W/paper_2310_03978_b200/libtn.so $ROOT/build_ab/libtn_B.so
git -C $ROOT worktree remove --force $W
echo "built $REV -> build_ab/libtn_B.so"
