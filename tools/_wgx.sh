python -m pytest tests/test_conv_gpu.py tests/test_unet_gpu.py -x -q 2>&1 | tail -2
for L in paper_2403_13135_b200/_C/base/libicelabel_b200.so paper_2403_13135_b200/_C/libicelabel_b200.so; do
ICE_LIB_PATH=$L python tools/time_halve.py 32 128 128 128 64
ICE_LIB_PATH=$L python tools/time_conv.py wgrad 32 256 256 64 0 64
ICE_LIB_PATH=$L python tools/time_conv.py wgrad 32 256 256 64 64 64
done
bash tools/ab_bench.sh paper_2403_13135_b200/_C/base/libicelabel_b200.so paper_2403_13135_b200/_C/libicelabel_b200.so 3
