O=gpurun_out/r02
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_determinism.py tests/test_gpu_edges.py tests/test_gpu_fullsize.py -m gpu -q -x --timeout 600 -p no:cacheprovider 2>&1 | tail -3
for c in cfg5 cfg3 cfg2; do
  timeout 300 python bench.py --config $c --no-extra --steps 20 > $O/bench_$c.json 2> $O/bench_$c.err
  python -c "import json; d=json.load(open('$O/bench_$c.json')); print('$c', d['ms_per_step'], d['kernels_ms'])"
done
