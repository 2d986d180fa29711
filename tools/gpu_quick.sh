#!/bin/bash
# Quick GPU iteration: selected GPU tests, a short bench, the per-call layer profile and the
# ncu launch list of two eager steps.
#   gpurun --timeout 1500 -- 'bash tools/gpu_quick.sh "tests/test_train_gpu.py tests/test_conv_gpu.py"'
mkdir -p gpurun_out
T=${1:-"tests/test_train_gpu.py tests/test_graph_gpu.py tests/test_conv_gpu.py"}
timeout 900 python -m pytest $T -q -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/tq.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1
timeout 300 python tools/profile_layers.py > gpurun_out/layers.txt 2>&1
if [ -z "$NO_NCU" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file gpurun_out/launches.csv python tools/profile_step.py --steps 2 > gpurun_out/launches.log 2>&1
fi
