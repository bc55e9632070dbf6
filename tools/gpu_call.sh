O=gpurun_out/r02
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_determinism.py tests/test_gpu_delta.py tests/test_gpu_rr.py tests/test_gpu_next4.py -m gpu -q --timeout 600 -p no:cacheprovider 2>&1 | tail -2
python tools/kxk_stamps.py 2>&1 | grep "k="
