# bench one config under several environment settings: CFG=cfg5 VAR=REFINE_ST_PF VALS="0 1 2 3" bash tools/sweep_env.sh
O=gpurun_out/sw
mkdir -p $O
for v in $VALS; do
  env $EXTRA $VAR=$v timeout 300 python bench.py --config $CFG --no-extra --steps ${STEPS:-20} > $O/b_${CFG}_$v.json 2> $O/b_${CFG}_$v.err
  python -c "import json; d=json.load(open('$O/b_${CFG}_$v.json')); print('$CFG $VAR=$v', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['kernels_ms'].items()})" || tail -3 $O/b_${CFG}_$v.err
done
