set -x
python -m pytest tests/test_gpu_parity.py tests/test_gpu_regimes.py -x -q -k "wide or lu or ilu or schwarz or c2analog or c3proxy" 2>&1 | tail -5
for nv in 1 0; do
ACCH_NARROW=$nv ACCH_DEBUG=1 python tools/precond_probe.py c2 c3 2>&1 | grep -E "^\{|precond:" | cut -c1-170
done
