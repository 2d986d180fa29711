#!/bin/bash
# Round-2 final evidence (under gpurun): ncu launch list of two warm train steps (time + DRAM
# bytes per launch) and full captures (--set full) of the top kernels of each class, incl.
# the round-2 kernels (deferred finisher batch, fused stem, max-pool backward) and K1.
#   gpurun --timeout 3600 -- 'bash tools/gpu_profiles_r02.sh'
mkdir -p gpurun_out
P=${P:-r02f}
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
[ -z "$ONLY" ] && timeout 900 ncu --metrics $M --clock-control none -c 3000 --csv --log-file gpurun_out/${P}_launches.csv \
  python tools/profile_step.py --steps 3 > gpurun_out/${P}_launches.log 2>&1
[ -z "$ONLY" ] && timeout 600 ncu --metrics $M --clock-control none -c 50 --csv --log-file gpurun_out/${P}_launches_al.csv \
  python tools/profile_autolabel.py > gpurun_out/${P}_launches_al.log 2>&1
F="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
cap() {  # name regex skip   (ONLY="a b": just those captures)
  if [ -n "$ONLY" ] && [[ " $ONLY " != *" $1 "* ]]; then return; fi
  timeout 600 $F -k "regex:$2" -s $3 -c 1 -o gpurun_out/${P}_$1 -f python tools/profile_step.py --steps 3 > gpurun_out/${P}_$1.log 2>&1
}
cap flush "flush_kernel" 2
cap stem_fprop "stem_fprop_kernel" 2
cap stem_wgrad "stem_wgrad_kernel" 2
cap maxpool_bwd0 "maxpool_bwd_kernel" 14
cap head "head_ce_kernel" 2
cap adam "adam_kernel" 2
cap wgrad_m2 "conv_gemm_m2<.int.256, .int.3, .*WgradProb" 40
cap halo_fp64 "halo_gemm<.int.64, .int.1, .bool.1, .*FpropProb" 2
cap halo_dg64 "halo_gemm<.int.64, .int.1, .bool.1, .*DgradProb" 2
cap halo_dg128 "halo_gemm<.int.128, .int.2, .bool.0, .*DgradProb" 2
cap halo_fp128 "halo_gemm<.int.128, .int.2, .bool.0, .*FpropProb" 6
cap halo_fp128p "halo_gemm<.int.128, .int.4, .bool.0, .*FpropProb" 4
cap halo_dg128p "halo_gemm<.int.128, .int.4, .bool.0, .*DgradProb" 2
cap halo_fp64p "halo_gemm<.int.64, .int.6, .bool.0, .*FpropProb" 2
cap hwgrad64 "hwgrad_kernel<.int.64, .int.2, .int.2, .bool.0" 2
cap fprop256 "conv_gemm<.int.256, .int.4, .*FpropProb" 20
[ -z "$ONLY" ] && timeout 600 $F -k "regex:autolabel256" -s 1 -c 1 -o gpurun_out/${P}_autolabel256 -f python tools/profile_autolabel.py --reps 1 > gpurun_out/${P}_al.log 2>&1
# summarise on the box and drop the reports (gpurun copies back at most 64 MiB); KEEP="a b"
# keeps those captures' .ncu-rep files
python tools/summarize_ncu_full.py gpurun_out/${P}_ncu_full_summary.json gpurun_out/${P}_*.ncu-rep > gpurun_out/${P}_summary.log 2>&1
for f in gpurun_out/${P}_*.ncu-rep; do
  n=${f#gpurun_out/${P}_}; n=${n%.ncu-rep}
  [[ " $KEEP " == *" $n "* ]] || rm -f "$f"
done
ls -la gpurun_out/ | tail -30
