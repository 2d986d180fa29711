# A/B of the coarse-group size of K1's two-level channel medians (builds under _C/v<cg>) + parity
mkdir -p gpurun_out
for v in base "$@"; do
  if [ $v = base ]; then unset ICE_LIB_PATH; else export ICE_LIB_PATH=$PWD/paper_2403_13135_b200/_C/v$v/libicelabel_b200.so; fi
  timeout 600 python -m pytest tests/test_autolabel_gpu.py -q -x -p no:cacheprovider -k "swar or batch or region_path_forced" 2>&1 | tail -1 | sed "s/^/cg=$v tests: /" >> gpurun_out/al_cg.log
  for k in tgray tint trand; do echo "cg=$v $(timeout 300 python tools/time_autolabel.py --tiles 14800 --kind $k 2>&1 | tail -1)" >> gpurun_out/al_cg.log; done
done
