# quick check: kernels touched by a change -> determinism / stencil / fullsize tests + cfg5 / cfg4 bench lines
O=gpurun_out/q
mkdir -p $O
timeout 900 python -m pytest ${TESTS:-tests/test_gpu_determinism.py tests/test_gpu_stencil.py} -m gpu -q -x --timeout 600 -p no:cacheprovider 2>&1 | tail -3
for c in ${CFGS:-cfg5 cfg4}; do
  timeout 300 python bench.py --config $c --no-extra --steps 20 > $O/bench_$c.json 2> $O/bench_$c.err
  python -c "import json; d=json.load(open('$O/bench_$c.json')); print('$c', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['kernels_ms'].items()})"
done
