set -x
python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -x -q 2>&1 | tail -4
python tools/res_bench.py --eps 1e-4
python tools/res_bench.py --eps 1e-3
python tools/res_bench.py --eps 0
python tools/run_configs.py --configs 2 --steps 30 --profile --out gpurun_out/j4 2>&1 | cut -c1-2000
ncu --set full --clock-control none --import-source on -k regex:res_zm -c 1 -o gpurun_out/r02_res_zm_v1 python tools/res_bench.py --once > gpurun_out/ncu_res.log 2>&1
ncu -i gpurun_out/r02_res_zm_v1.ncu-rep --page raw --csv --metrics smsp__inst_executed.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active 2>&1 | tail -3
