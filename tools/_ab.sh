python -m pytest tests/test_conv_gpu.py tests/test_unet_gpu.py -x -q 2>&1 | tail -3
bash tools/ab_env.sh ICE_WG_M2=0 3
