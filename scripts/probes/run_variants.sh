# run_variants.sh "<codec gradset> ..." v1 v2 ... : one compact bench line per (variant, case)
cases=$1; shift
cp paper_2103_15195_b200/libmergecomp.so /tmp/default.so
for v in "$@"; do
  cp gpurun_variants/$v.so paper_2103_15195_b200/libmergecomp.so
  for cg in $cases; do c=${cg%%:*}; g=${cg##*:}; echo -n "$v "; bash scripts/codec_line.sh $c $g; done
done
cp /tmp/default.so paper_2103_15195_b200/libmergecomp.so
