#!/bin/bash
# Steady-state DRAM traffic per launch of K1 and the selection kernel (no cache flush between
# launches: --cache-control none; only the dram__bytes / duration metrics, so the kernels replay
# without state changes): consecutive eager steps of the bench workload (tools/prof_step.py).
# Usage (on the GPU box): tools/k1_traffic.sh OUT.csv
set -e
cd "$(dirname "$0")/.."
out=${1:-gpurun_out/k1_traffic.csv}
python tools/prof_step.py --steps 120 > /dev/null
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --cache-control none \
    --clock-control none -k regex:"accum_emit|select_kernel" -s 200 -c 20 --csv --log-file "$out" \
    python tools/prof_step.py --steps 120 > /dev/null
