#!/bin/bash
# Roofline denominators (peaks.cu) on one B200 with nvidia-smi clock / throttle samples alongside.
# Output: gpurun_out/peaks.jsonl (one line per kernel) + gpurun_out/peaks_clocks.csv
cd "$(dirname "$0")"
OUT=../../gpurun_out
mkdir -p $OUT
[ -x peaks ] || nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o peaks peaks.cu
nvidia-smi --query-gpu=timestamp,index,clocks.sm,clocks.max.sm,power.draw,power.limit,temperature.gpu,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 100 > $OUT/peaks_clocks.csv &
SMI=$!
./peaks > $OUT/peaks.jsonl 2>&1
RC=$?
kill $SMI
cat $OUT/peaks.jsonl
exit $RC
