# build libmergecomp.so variants for A/B runs: build_variants.sh name "flags" [name "flags" ...]
# outputs gpurun_variants/<name>.so (git-ignored, travels with gpurun); restores the default build
set -e
mkdir -p gpurun_variants
while [ $# -ge 2 ]; do
  MC_NVCC_EXTRA="$2" python -m paper_2103_15195_b200.build --force > /dev/null
  cp paper_2103_15195_b200/libmergecomp.so gpurun_variants/$1.so
  echo "built $1 ($2)"
  shift 2
done
python -m paper_2103_15195_b200.build --force > /dev/null
