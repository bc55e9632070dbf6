O=gpurun_out/r02
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_determinism.py tests/test_gpu_delta.py tests/test_gpu_edges.py tests/test_gpu_mixed.py -m gpu -q --timeout 600 -p no:cacheprovider > $O/pytest_14.txt 2>&1
tail -2 $O/pytest_14.txt; grep -E "^FAILED" $O/pytest_14.txt | head
python tools/kxk_stamps.py 2>&1 | grep "k=" 
for c in cfg3 cfg5; do
  timeout 300 python bench.py --config $c --no-extra --steps 5 > $O/bench_$c.json 2> $O/bench_$c.err
  python -c "import json; d=json.load(open('$O/bench_$c.json')); print('$c', d['ms_per_step'], d['kernels_ms']['kxk_finish'])"
done
