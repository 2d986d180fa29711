# A/B of the coarse-group size of K1's two-level channel medians (builds under _C/v<cg>)
mkdir -p gpurun_out
for v in base 4 6 12 16; do
  if [ $v = base ]; then unset ICE_LIB_PATH; else export ICE_LIB_PATH=$PWD/paper_2403_13135_b200/_C/v$v/libicelabel_b200.so; fi
  for k in tgray tint trand; do echo "cg=$v $(timeout 300 python tools/time_autolabel.py --tiles 14800 --kind $k 2>&1 | tail -1)" >> gpurun_out/al_cg.log; done
done
