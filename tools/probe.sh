#!/bin/bash
# One-off box probe: host cores, GPU, FP64 rates.
mkdir -p gpurun_out
{ nproc; lscpu | head -20; nvidia-smi; python -c "import os; print('cpu_count', os.cpu_count(), 'affinity', len(os.sched_getaffinity(0)))"; ./tools/fp64_probe; } > gpurun_out/probe.txt 2>&1
cat gpurun_out/probe.txt
