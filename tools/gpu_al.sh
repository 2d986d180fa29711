mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_autolabel_gpu.py tests/test_native_abi.py -q -p no:cacheprovider -x > gpurun_out/al_tests.log 2>&1; echo "exit $?" >> gpurun_out/al_tests.log
for k in tgray tint trand; do timeout 300 python tools/time_autolabel.py --size 512 --tiles 2960 --uniq 74 --kind $k >> gpurun_out/al_time.log 2>&1; done
timeout 300 python tools/time_autolabel.py --tiles 14800 --kind tgray >> gpurun_out/al_time.log 2>&1
timeout 300 python tools/time_autolabel.py --tiles 14800 --kind tgray --path 3 >> gpurun_out/al_time.log 2>&1
