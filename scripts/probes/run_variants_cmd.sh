# run_variants_cmd.sh "<command>" v1 v2 ... : run a command under each library variant
cmd=$1; shift
cp paper_2103_15195_b200/libmergecomp.so /tmp/default.so
for v in "$@"; do
  cp gpurun_variants/$v.so paper_2103_15195_b200/libmergecomp.so
  echo "== $v"; bash -c "$cmd"
done
cp /tmp/default.so paper_2103_15195_b200/libmergecomp.so
