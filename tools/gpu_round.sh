#!/bin/bash
# One GPU call: GPU tests, the bench line, the ncu launch list and full captures.
#   gpurun --timeout 3000 -- 'bash tools/gpu_round.sh [tests] [bench] [launches] [full] [al]'
set -x
mkdir -p gpurun_out
want() { [ -z "$STAGES" ] || [[ " $STAGES " == *" $1 "* ]]; }
STAGES="$*"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt 2>&1
if want tests; then
  timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
  echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
  tail -3 gpurun_out/pytest_gpu.log
fi
if want smoke; then
  timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
fi
if want bench; then
  timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?"
  cat gpurun_out/bench.json
fi
if want launches; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file gpurun_out/launches.csv python tools/profile_step.py --steps 2 > gpurun_out/launches.log 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 50 --csv \
    --log-file gpurun_out/launches_al.csv python tools/profile_autolabel.py > gpurun_out/launches_al.log 2>&1
fi
if want full; then
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:conv_gemm -s 60 -c 4 \
    -o gpurun_out/prof_conv -f python tools/profile_step.py --steps 2 > gpurun_out/prof_conv.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:halo_gemm -s 8 -c 3 \
    -o gpurun_out/prof_halo -f python tools/profile_step.py --steps 2 > gpurun_out/prof_halo.log 2>&1
fi
if want al; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"autolabel_kernel|segment_vec" -s 1 -c 2 \
    -o gpurun_out/prof_al -f python tools/profile_autolabel.py --reps 1 > gpurun_out/prof_al.log 2>&1
fi
ls -la gpurun_out
