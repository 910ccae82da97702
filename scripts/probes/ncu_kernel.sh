# usage: ncu_kernel.sh <name> <kernel-regex> <bench args...> : one ncu --set full capture
name=$1; kre=$2; shift 2
ncu --set full --clock-control none --import-source on -k regex:$kre -c 1 -f -o gpurun_out/$name python bench.py --steps 1 --warmup 1 --no-search --no-cpu-baseline --e2e-steps 1 "$@" > gpurun_out/$name.log 2>&1
