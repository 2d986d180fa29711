timeout 300 python -m pytest tests/test_conv_gpu.py -x -q -k wgrad 2>&1 | tail -3 || exit 1
for sh in "32 16 16 1024 0 1024" "32 32 32 512 0 512" "32 64 64 256 256 256" "32 16 16 1024 1024 1024" "32 8 8 2048 0 2048" "32 8 8 1024 0 2048"; do
 for m in 0 1; do echo -n "pair=$m "; ICE_WG_PAIR=$m timeout 60 python tools/time_conv.py wgrad $sh; done
done
timeout 600 python -m pytest tests/test_conv_gpu.py tests/test_unet_gpu.py -x -q 2>&1 | tail -2
bash tools/ab_env.sh ICE_WG_PAIR=0 2
