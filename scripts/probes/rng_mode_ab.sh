set -x
export MC_RNG_MODE=2
python -m pytest tests/test_gpu_codecs.py tests/test_gpu_configs.py tests/test_gpu_sync.py -m gpu -x -q -k "qsgd or terngrad or c3 or rng or quantizer" 2>&1 | tail -5
for m in 0 2; do
  export MC_RNG_MODE=$m
  for c in qsgd terngrad; do for gs in resnet50_161 resnet101_314; do echo "mode=$m"; bash scripts/codec_line.sh $c $gs; done; done
done
