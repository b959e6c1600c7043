timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_regimes.py -x -q -k "wide or lu or ilu or schwarz or c2analog or c3proxy" 2>&1 | tail -3
timeout 120 python tools/precond_probe.py c2 c3 2>&1 | grep -E "^\{" | cut -c1-140
