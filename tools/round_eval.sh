set -x
mkdir -p gpurun_out/r01
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/r01/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r01/smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/r01/bench.json 2> gpurun_out/r01/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r01/reference.json 2> gpurun_out/r01/reference.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01/launches_cfg3.csv python bench.py --config cfg3 --steps 2 --warmup 3 --no-extra > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01/launches_cfg5.csv python bench.py --config cfg5 --steps 2 --warmup 3 --no-extra > /dev/null 2>&1
timeout 600 ncu --set full --import-source on -k regex:gemm_ax -c 1 -o gpurun_out/r01/full_cfg3_gemm python bench.py --config cfg3 --steps 1 --warmup 3 --no-extra > /dev/null 2>&1
timeout 600 ncu --set full --import-source on -k regex:"spmm_gather|passB_kernel" -c 2 -o gpurun_out/r01/full_cfg4 python bench.py --config cfg4 --steps 1 --warmup 3 --no-extra > /dev/null 2>&1
timeout 600 ncu --set full --import-source on -k regex:"passB2_kernel|spmm_gather|passC" -c 3 -o gpurun_out/r01/full_cfg5 python bench.py --config cfg5 --steps 1 --warmup 3 --no-extra > /dev/null 2>&1
ls -la gpurun_out/r01
cat gpurun_out/r01/pytest_gpu.txt gpurun_out/r01/smoke.txt
