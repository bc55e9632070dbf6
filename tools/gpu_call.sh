O=gpurun_out/r02
mkdir -p $O
for w in 1 2 4; do
  REFINE_WF_PER_SM=$w timeout 300 python bench.py --config cfg3 --no-extra --steps 10 > $O/bench_cfg3.json 2> $O/bench_cfg3.err
  python -c "import json; d=json.load(open('$O/bench_cfg3.json')); print('wf=$w cfg3', d['ms_per_step'], d['kernels_ms']['w_finish'], d['kernels_ms']['kxk_rq'])"
done
