set -x
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 200 python tools/precond_probe.py c2 c3 2>&1 | grep -E "^\{" | cut -c1-150
