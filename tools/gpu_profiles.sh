#!/bin/bash
# Round-end profiling: ncu launch list (time + DRAM bytes) of the bench command and full
# captures of the top kernels.  Usage (under gpurun): bash tools/gpu_profiles.sh
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 4000 --csv \
  --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-autolabel --no-cpu --no-config5 --corpus 1024 \
  > gpurun_out/launches_bench.log 2>&1
K="--kernel-name-base demangled"
timeout 600 ncu --set full --clock-control none --import-source on $K -k "regex:hwgrad_kernel<.int.64, .int.2" -s 1 -c 1 \
  -o gpurun_out/full_hwgrad64 -f python tools/profile_step.py --steps 2 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on $K -k "regex:conv_gemm_m2<.int.256, .int.3, .*WgradProb" -s 10 -c 2 \
  -o gpurun_out/full_wgrad_m2 -f python tools/profile_step.py --steps 2 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on $K -k "regex:conv_gemm_m2<.int.256, .int.3, .*DgradProb" -s 2 -c 1 \
  -o gpurun_out/full_dgrad_m2 -f python tools/profile_step.py --steps 2 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on $K -k "regex:halo_gemm<.int.64, .int.1, .bool.1.*FpropProb" -s 2 -c 1 \
  -o gpurun_out/full_halo_fp64 -f python tools/profile_step.py --steps 2 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on $K -k "regex:halo_gemm<.int.64, .int.1, .bool.1.*DgradProb" -s 2 -c 1 \
  -o gpurun_out/full_halo_dg64 -f python tools/profile_step.py --steps 2 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on $K -k "regex:autolabel256" -s 1 -c 1 \
  -o gpurun_out/full_autolabel256 -f python tools/profile_autolabel.py --reps 1 > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
