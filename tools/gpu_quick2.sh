# targeted GPU tests (args: pytest -k expression or files) + bench line
mkdir -p gpurun_out
timeout 1500 python -m pytest $TESTS -q -x -p no:cacheprovider > gpurun_out/quick_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/quick_tests.log
if [ -n "$BENCH" ]; then timeout 900 python bench.py $BENCH > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?" >> gpurun_out/quick_tests.log; fi
