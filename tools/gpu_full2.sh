#!/bin/bash
# ncu --set full captures of single launches of the step's top kernels (one report each, small
# enough for gpurun_out), from step 3 of tools/profile_step.py.
mkdir -p gpurun_out
cap() {  # name regex skip
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:$2" -s "$3" -c 1 -o "gpurun_out/r02_$1" -f python tools/profile_step.py --steps 3 > "gpurun_out/r02_$1.log" 2>&1
}
cap wgrad_m2 "conv_gemm_m2<.int.256.*WgradProb" 40
cap halo_fp64 "halo_gemm<.int.64, .int.1, .bool.1, .*FpropProb" 5
cap halo_dg64 "halo_gemm<.int.64, .int.1, .bool.1, .*DgradProb" 5
cap halo_dg128 "halo_gemm<.int.128.*DgradProb" 10
cap hwgrad64 "hwgrad_kernel<.int.64, .int.1, .int.6" 5
cap hwgrad_cat "hwgrad_kernel<.int.64, .int.2, .int.3, .bool.0" 3
cap fprop256 "conv_gemm<.int.256, .int.4, .*FpropProb" 30
du -sh gpurun_out
