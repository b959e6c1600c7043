set -x
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_gpu_regimes.py -x -q -k "chord or residual or dvd or jacobian or c4analog or newton" 2>&1 | tail -3
for e in 1e-4 1e-3 0; do timeout 120 python tools/res_bench.py --eps $e | tail -1; done
