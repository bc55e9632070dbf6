O=gpurun_out/r02
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_delta.py tests/test_gpu_edges.py -m gpu -q --timeout 600 -p no:cacheprovider > $O/pytest_7.txt 2>&1
tail -2 $O/pytest_7.txt; grep -E "^FAILED" $O/pytest_7.txt | head
for t in 0 1; do
for c in cfg3 cfg2; do
  REFINE_GEMM_TMA=$t timeout 300 python bench.py --config $c --no-extra --steps 10 > $O/bench_$c.json 2> $O/bench_$c.err
  python -c "import json; d=json.load(open('$O/bench_$c.json')); print('tma=$t $c', d['ms_per_step'], d.get('kernels_ms',{}).get('gemm_ax'), d['roofline']['frac'] if d.get('roofline') else None)"
done
done
