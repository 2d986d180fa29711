timeout 600 python -m pytest tests/test_conv_gpu.py -x -q 2>&1 | tail -2
for m in 0 1; do echo -n "m2=$m "; ICE_CONV_M2=$m timeout 60 python tools/time_conv.py dgrad 32 64 64 128 0 256; done
for m in 0 1; do echo -n "m2=$m "; ICE_CONV_M2=$m timeout 60 python tools/time_conv.py dgrad 32 32 32 128 0 256; done
timeout 600 python -m pytest tests/test_unet_gpu.py tests/test_graph_gpu.py -x -q 2>&1 | tail -2
python tools/profile_layers.py > gpurun_out/layers7.txt 2>&1
ICE_LIB_PATH=paper_2403_13135_b200/_C/base/libicelabel_b200.so python tools/profile_layers.py > gpurun_out/layers7_base.txt 2>&1
bash tools/ab_bench.sh paper_2403_13135_b200/_C/base/libicelabel_b200.so paper_2403_13135_b200/_C/libicelabel_b200.so 3
