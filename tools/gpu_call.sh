O=gpurun_out/r02
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next3.py tests/test_gpu_next4.py tests/test_gpu_rr.py tests/test_gpu_edges.py tests/test_gpu_mixed.py tests/test_gpu_emul.py -m gpu -q --timeout 600 -p no:cacheprovider > $O/pytest_9.txt 2>&1
tail -2 $O/pytest_9.txt; grep -E "^FAILED|Error" $O/pytest_9.txt | head
