# qsgd / terngrad parity subset + bench lines (R50, R101)
python -m pytest tests/test_gpu_codecs.py tests/test_gpu_configs.py tests/test_gpu_sync.py -m gpu -x -q -k "qsgd or terngrad or c3 or rng or quantizer" 2>&1 | tail -3
for c in qsgd terngrad; do for gs in resnet50_161 resnet101_314; do bash scripts/codec_line.sh $c $gs; done; done
