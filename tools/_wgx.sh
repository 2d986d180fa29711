python -m pytest tests/ -x -q -m gpu -k "head or unet or graph or train" 2>&1 | tail -2
python tools/profile_layers.py | grep -E "head_ce|total"
ICE_LIB_PATH=paper_2403_13135_b200/_C/base/libicelabel_b200.so python tools/profile_layers.py | grep -E "head_ce|total"
bash tools/ab_bench.sh paper_2403_13135_b200/_C/base/libicelabel_b200.so paper_2403_13135_b200/_C/libicelabel_b200.so 2
