timeout 600 python -m pytest tests/test_unet_gpu.py tests/test_graph_gpu.py -x -q 2>&1 | tail -2
timeout 600 python -m pytest tests/ -x -q -m gpu -k "pool" 2>&1 | tail -2
python tools/profile_layers.py | grep -E "maxpool_bwd|total"
ICE_LIB_PATH=paper_2403_13135_b200/_C/base/libicelabel_b200.so python tools/profile_layers.py | grep -E "maxpool_bwd|total"
bash tools/ab_bench.sh paper_2403_13135_b200/_C/base/libicelabel_b200.so paper_2403_13135_b200/_C/libicelabel_b200.so 2
