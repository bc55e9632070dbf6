O=gpurun_out/r02
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_determinism.py -m gpu -q --timeout 600 -p no:cacheprovider > $O/pytest_det.txt 2>&1
tail -3 $O/pytest_det.txt; grep -E "^FAILED" $O/pytest_det.txt
