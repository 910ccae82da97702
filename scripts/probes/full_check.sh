# full GPU suite + smoke + default bench + codec sweeps (R50, Mask R-CNN) + launch lists
python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/full_gputest.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/full_smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/full_smoke.txt
python bench.py > gpurun_out/full_bench.log 2>&1
python bench.py --impl reference > gpurun_out/full_bench_ref.log 2>&1
for gs in resnet50_161 maskrcnn_201 resnet101_314 vgg16_32; do echo "== $gs"; bash scripts/sweep_codecs.sh $gs; done > gpurun_out/full_sweep.txt 2>&1
bash scripts/launch_list.sh resnet50_161 efsignsgd onebit int8 qsgd terngrad dgc_lite topk randk threshold signsgd signum fp16 identity > gpurun_out/full_launch_lists.txt 2>&1
