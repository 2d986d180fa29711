bash tools/gpu_round.sh tests smoke bench > gpurun_out/round.log 2>&1
bash tools/gpu_profiles.sh > gpurun_out/profiles.log 2>&1
