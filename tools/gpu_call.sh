O=gpurun_out/r02
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_delta.py tests/test_gpu_determinism.py tests/test_gpu_edges.py tests/test_gpu_next3.py tests/test_gpu_next4.py tests/test_gpu_rr.py tests/test_gpu_accuracy.py tests/test_gpu_stencil.py -m gpu -q --timeout 600 -p no:cacheprovider > $O/pytest_11.txt 2>&1
tail -2 $O/pytest_11.txt; grep -E "^FAILED" $O/pytest_11.txt | head
for t in 1 0; do
for c in cfg1 cfg2; do
  REFINE_TAIL=$t timeout 300 python bench.py --config $c --no-extra --steps 20 > $O/bench_$c.json 2> $O/bench_$c.err
  python -c "import json; d=json.load(open('$O/bench_$c.json')); print('tail=$t $c', round(d['ms_per_step']*1000,1), 'us', d['kernels_ms'])"
done
done
