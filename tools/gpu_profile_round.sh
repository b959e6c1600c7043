#!/bin/bash
# One GPU session: bench (JSON line) on the driver's command, the reference
# arm, the ncu launch list of the bench's workload, and one `ncu --set full`
# capture per hot kernel (tools/micro.py at 256^3; the column-sweep solver on
# BASELINE configs 2 and 3 through tools/precond_probe.py).  Reports are
# written to /tmp on the box and summarised there; only summaries and the
# small reports come back in gpurun_out/ (64 MiB cap).
# Usage (on the GPU box, from the repo root): bash tools/gpu_profile_round.sh TAG
set -u
TAG=${1:-v}
OUT=gpurun_out
TMP=/tmp/prof_$TAG
mkdir -p $OUT $TMP
if [ -z "${NOBENCH:-}" ]; then
  timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $OUT/bench_${TAG}_W5K20.json 2> $OUT/bench_${TAG}_W5K20.err
  timeout 900 python bench.py > $OUT/bench_${TAG}_W3K4.json 2> $OUT/bench_${TAG}_W3K4.err
  timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $OUT/bench_${TAG}_ref_W5K20.json 2> $OUT/bench_${TAG}_ref.err
fi
# the launch list runs the bench's workload with K=1 timed step and no e2e
# replay (the full command's ~70k launches take over half an hour under ncu)
if [ -z "${NOLAUNCH:-}" ]; then
  timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $TMP/launches.csv \
      python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > $OUT/bench_ncu_$TAG.log 2>&1
  python tools/ncu_summary.py $TMP/launches.csv > $OUT/launches_${TAG}_summary.txt
  gzip -c $TMP/launches.csv > $OUT/launches_$TAG.csv.gz
fi
for k in apply_group lagupd_dev mdot_grouped mv_zm res_zm factor_kernel; do
  name=$(echo "$k" | tr -c 'a-z0-9_\n' '_')
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"$k" -s 2 -c 1 \
      -o $TMP/${TAG}_full_$name python tools/micro.py > $OUT/ncu_${TAG}_$name.log 2>&1
done
for c in c2 c3; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:apply_cols -s 2 -c 1 \
      -o $TMP/${TAG}_full_apply_cols_$c python tools/precond_probe.py $c > $OUT/ncu_${TAG}_apply_cols_$c.log 2>&1
done
python tools/ncu_full_summary.py $TMP/*.ncu-rep > $OUT/ncu_full_${TAG}_summary.txt
python tools/ncu_traffic.py $TMP/*.ncu-rep > $OUT/traffic_$TAG.json
for name in apply_group mv_zm res_zm apply_cols_c2 apply_cols_c3; do
  for f in $TMP/${TAG}_full_${name}*.ncu-rep; do
    python tools/ncu_stalls.py $f 30 > $OUT/stalls_${TAG}_$name.txt
  done
done
ls -la $OUT
