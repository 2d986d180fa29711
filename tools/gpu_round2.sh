#!/bin/bash
# Round-2 evidence run: GPU tests, smoke, bench, the ncu launch list of the bench step and
# full captures of the top kernels (tcgen05 metrics), K1 launch list + full capture.
#   gpurun --timeout 3600 -- 'bash tools/gpu_round2.sh [tests] [bench] [launches] [full] [al]'
mkdir -p gpurun_out
want() { [ -z "$STAGES" ] || [[ " $STAGES " == *" $1 "* ]]; }
STAGES="$*"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt 2>&1
if want tests; then
  timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
  echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
  timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
fi
if want bench; then
  timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?"
fi
if want launches; then
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv \
    --log-file gpurun_out/launches.csv python tools/profile_step.py --steps 2 > gpurun_out/launches.log 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 50 --csv \
    --log-file gpurun_out/launches_al.csv python tools/profile_autolabel.py > gpurun_out/launches_al.log 2>&1
fi
if want full; then
  # step 3 of profile_step (warm): the m2 wgrad, the level-0 halo fprop / dgrad, the level-0 hwgrad
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"conv_gemm|halo_gemm|hwgrad|head_ce|adam|colsum|splitsum" -s 180 -c 90 \
    -o gpurun_out/r02_full_step -f python tools/profile_step.py --steps 3 > gpurun_out/prof_step.log 2>&1
fi
if want al; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"autolabel256" -s 1 -c 1 \
    -o gpurun_out/r02_full_al -f python tools/profile_autolabel.py --reps 1 > gpurun_out/prof_al.log 2>&1
fi
ls -la gpurun_out | tail -20
