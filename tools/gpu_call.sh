O=gpurun_out/r02
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next4.py tests/test_gpu_emul.py tests/test_gpu_accuracy.py -m gpu -q --timeout 600 -p no:cacheprovider -x > $O/pytest_6.txt 2>&1
tail -3 $O/pytest_6.txt; grep -E "^FAILED|Error" $O/pytest_6.txt | head
