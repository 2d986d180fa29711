set -x
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 4000 --csv \
    --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-autolabel --no-cpu --no-config5 --corpus 1024 > gpurun_out/launches_bench.log 2>&1
tail -2 gpurun_out/launches_bench.log
