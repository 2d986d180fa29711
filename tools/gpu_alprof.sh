# K1 phase profile (clock64 marks) on T-gray / T-tint / T-rand
mkdir -p gpurun_out
export ICE_LIB_PATH=$PWD/paper_2403_13135_b200/_C/prof/libicelabel_b200.so
for k in tgray tint trand; do timeout 300 python tools/time_autolabel.py --tiles 2960 --kind $k --prof >> gpurun_out/al_prof.log 2>&1; done
