O=gpurun_out/r02
mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"passB2_tma|passC_kernel" -c 2 -f -o $O/pb_cfg5 python bench.py --config cfg5 --steps 1 --warmup 3 --no-extra > /dev/null 2>&1
python tools/ncu_summary.py report $O/pb_cfg5.ncu-rep $O/ncu_pb_cfg5.json > /dev/null
ls -la $O/pb_cfg5.ncu-rep
