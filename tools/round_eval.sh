# Round-end evidence: GPU tests, smoke, bench (+ reference arm), ncu launch lists and full captures.
#   gpurun --timeout 3600 -- 'bash tools/round_eval.sh'
set -x
O=gpurun_out/${EVAL_TAG:-r02}
mkdir -p $O
[ -n "$SKIP_TESTS" ] || timeout 1700 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider 2>&1 | tail -5 > $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > $O/reference.json 2> $O/reference.err
K="gemm_ax|w_finish|kxk_|passB|passC|spmm_|norm|ag_local"
for c in cfg1 cfg3 cfg4 cfg5; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"$K" -c 200 --csv --log-file $O/launches_$c.csv \
    python bench.py --config $c --steps 2 --warmup 3 --no-extra > /dev/null 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_ax -c 1 -o $O/full_cfg3_gemm \
  python bench.py --config cfg3 --steps 1 --warmup 3 --no-extra > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"spmm_stencil|spmm_gather|passB_kernel|passC_kernel|kxk_finish" -c 4 \
  -o $O/full_cfg4 python bench.py --config cfg4 --steps 1 --warmup 3 --no-extra > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"passB2|spmm_stencil|passC|kxk_finish" -c 6 \
  -o $O/full_cfg5 python bench.py --config cfg5 --steps 1 --warmup 3 --no-extra > /dev/null 2>&1
ls -la $O
cat $O/pytest_gpu.txt $O/smoke.txt
for c in cfg1 cfg3 cfg4 cfg5; do python tools/ncu_summary.py launches $O/launches_$c.csv $O/launches_$c.json > /dev/null; done
python tools/ncu_summary.py report $O/full_cfg3_gemm.ncu-rep $O/ncu_gemm_cfg3.json > /dev/null
python tools/ncu_summary.py report $O/full_cfg4.ncu-rep $O/ncu_cfg4.json > /dev/null
python tools/ncu_summary.py report $O/full_cfg5.ncu-rep $O/ncu_cfg5.json > /dev/null
[ -n "$KEEP_REPS" ] || rm -f $O/*.ncu-rep
head -c 1500 $O/bench.json
