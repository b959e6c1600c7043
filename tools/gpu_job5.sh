# round-2 session 3, job 1: tests at HEAD + smoke + preconditioner sweep (GMRES/step vs subdomain solver)
set -x
mkdir -p gpurun_out/s3
python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/s3/pytest_gpu.log
cat gpurun_out/s3/pytest_gpu.log
python __graft_entry__.py smoke 2>&1 | tail -2
for cfg in "8 ilu0 1" "8 ilu1 1" "8 ilu2 1" "8 ilu0 2" "8 ilu1 2" "16 ilu1 1" "16 ilu2 1" "4 ilu0 1" "4 lu 1"; do
  set -- $cfg
  timeout 600 python bench.py --n 128 --box $1 --solver $2 --overlap $3 --steps 4 --warmup 3 --no-e2e --no-cpu --verbose \
      > gpurun_out/s3/sweep128_box$1_$2_ov$3.json 2> gpurun_out/s3/sweep128_box$1_$2_ov$3.err
  grep -E "precond:|group solver|timed step|warmup step" gpurun_out/s3/sweep128_box$1_$2_ov$3.err | cut -c1-200
  python - <<PY
import json
try:
    d=json.load(open("gpurun_out/s3/sweep128_box$1_$2_ov$3.json"))
    k=d["kernels"]
    print("SWEEP $cfg", d["value"], d["solver_stats"]["per_step"], {n:(round(v["ms"]/max(v["launches"],1),3)) for n,v in k.items()})
except Exception as e:
    print("SWEEP $cfg failed", e)
PY
done
