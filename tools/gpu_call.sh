O=gpurun_out/r02
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > $O/pytest_13.txt 2>&1
tail -2 $O/pytest_13.txt; grep -E "^FAILED" $O/pytest_13.txt | head
