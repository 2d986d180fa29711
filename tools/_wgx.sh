ICE_LIB_PATH=paper_2403_13135_b200/_C/base/libicelabel_b200.so timeout 300 python -m pytest tests/test_conv_gpu.py -x -q -k stem 2>&1 | tail -2
timeout 300 python -m pytest tests/test_conv_gpu.py -x -q -k stem 2>&1 | tail -2
timeout 600 python -m pytest tests/test_unet_gpu.py tests/test_graph_gpu.py -x -q 2>&1 | tail -2
python tools/profile_layers.py | grep -E "stem|total"
ICE_LIB_PATH=paper_2403_13135_b200/_C/base/libicelabel_b200.so python tools/profile_layers.py | grep -E "stem|total"
