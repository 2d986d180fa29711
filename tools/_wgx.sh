python tools/profile_layers.py > gpurun_out/layers6.txt 2>&1
ICE_CONV_M2=0 python tools/profile_layers.py > gpurun_out/layers6_off.txt 2>&1
bash tools/ab_env.sh ICE_CONV_M2=0 3
