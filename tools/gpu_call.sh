# scratch GPU call (round 2): full GPU suite + default bench
O=gpurun_out/r02
mkdir -p $O
nproc > $O/nproc.txt
timeout 1700 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -rs --durations=20 -s > $O/pytest_gpu_1.txt 2>&1
tail -30 $O/pytest_gpu_1.txt
timeout 600 python bench.py > $O/bench_1.json 2> $O/bench_1.err
cat $O/bench_1.json | head -c 600
