set -x
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 120 python tools/precond_probe.py c2 c3 2>&1 | grep -E "^\{" | cut -c1-150
timeout 900 python tools/run_configs.py --configs 1,2,3 --profile --out gpurun_out/s3cfg 2>&1 | cut -c1-400 | tail -6
