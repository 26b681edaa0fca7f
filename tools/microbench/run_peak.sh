#!/bin/bash
# Runs the FP64 peak microbenchmark on a B200 with clock sampling.
cd "$(dirname "$0")"
mkdir -p ../../gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > ../../gpurun_out/peak_clocks.csv &
SMI=$!
./fp64_peak > ../../gpurun_out/fp64_peak.json 2>&1
kill $SMI
nvidia-smi > ../../gpurun_out/nvidia_smi.txt
lscpu > ../../gpurun_out/lscpu.txt
cat ../../gpurun_out/fp64_peak.json
