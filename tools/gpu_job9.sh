set -x
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_final_W5K20.json 2> gpurun_out/bench_final_W5K20.err
tail -c 600 gpurun_out/bench_final_W5K20.json
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_final_ref.json 2> gpurun_out/bench_final_ref.err
tail -c 1500 gpurun_out/bench_final_ref.json
